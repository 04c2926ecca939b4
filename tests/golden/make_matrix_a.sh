#!/usr/bin/env bash
# Regenerates tests/golden/matrix_a.json from the reference's own frozen
# golden vectors (proj/tests/oracle_data.hpp). Run in the build container,
# where /root/reference exists; the JSON is committed so the GPU box (which
# has no /root/reference) can use it.
set -euo pipefail
REF=${REF:-/root/reference/proj}
HERE=$(cd "$(dirname "$0")" && pwd)
TMP=$(mktemp -d)
cat > "$TMP/dump.cpp" <<'CPP'
#include <cstdio>
#include <string>
#include <vector>
#include "oracle_data.hpp"
template <class T> void arr(const char* name, const std::vector<T>& v, bool last = false) {
  std::printf("  \"%s\": [", name);
  for (size_t i = 0; i < v.size(); ++i) std::printf(i ? ", %s" : "%s", std::to_string(v[i]).c_str());
  std::printf("]%s\n", last ? "" : ",");
}
int main() {
  std::printf("{\n  \"source\": \"proj/tests/oracle_data.hpp\",\n");
  std::printf("  \"rows\": %lld, \"cols\": %lld,\n", (long long)oracle::rows_a, (long long)oracle::cols_a);
  std::vector<double> dense;
  for (auto& r : oracle::dense_a) for (double v : r) dense.push_back(v);
  arr("dense_a", dense);
  arr("coo_d0", oracle::coo_d0); arr("coo_d1", oracle::coo_d1); arr("coo_val", oracle::coo_val);
  arr("csr_ptr", oracle::csr_ptr); arr("csr_idx", oracle::csr_idx); arr("csr_val", oracle::csr_val);
  arr("ell_idx", oracle::ell_idx); arr("ell_val", oracle::ell_val);
  arr("ell_slot_of_entry", oracle::ell_slot_of_entry);
  arr("bcsr_ptr", oracle::bcsr_ptr); arr("bcsr_idx", oracle::bcsr_idx); arr("bcsr_val", oracle::bcsr_val);
  arr("row_nnz", oracle::row_nnz);
  arr("spmv_y", oracle::spmv_y);
  std::printf("  \"plan_coo_to_csr\": [");
  for (size_t i = 0; i < oracle::plan_coo_to_csr.size(); ++i)
    std::printf(i ? ", \"%s\"" : "\"%s\"", oracle::plan_coo_to_csr[i].c_str());
  std::printf("],\n  \"storage_explain\": {");
  bool first = true;
  for (const char* k : {"COO", "CSR", "CSC", "DCSR", "BCSR", "ELL"}) {
    std::printf("%s\"%s\": \"%s\"", first ? "" : ", ", k, oracle::storage_explain.at(k).c_str());
    first = false;
  }
  std::printf("}\n}\n");
}
CPP
g++ -std=c++20 -I"$REF/tests" -o "$TMP/dump" "$TMP/dump.cpp"
"$TMP/dump" > "$HERE/matrix_a.json"
rm -rf "$TMP"
echo "wrote $HERE/matrix_a.json"
