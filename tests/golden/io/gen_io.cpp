// Golden outputs of the reference's io.hpp text utilities (write_matrix_market,
// write_vector_text, read_tns incl. its error messages), for
// tests/cpp/test_io.cpp. Built against the unmodified reference headers by
// make_io_golden.sh; the outputs are committed next to this file.
#include <cstdio>
#include <fstream>
#include <iostream>

#include "sparseforge/io.hpp"
#include "sparseforge/tensor.hpp"

using namespace sparseforge;

int main(int argc, char** argv) {
  const std::string dir = argc > 1 ? argv[1] : ".";
  CooData d;
  d.shape.extents = {4, 5};
  d.coords = {{0, 1, 3, 3, 2}, {4, 0, 2, 3, 1}};
  d.values = {0.1, -2.5, 1.0 / 3.0, 6.02214076e23, 1e-300};
  write_matrix_market(dir + "/ref_out.mtx", d);
  write_vector_text(dir + "/ref_vec.txt", {0.1, -0.0, 3.0, 1.0 / 7.0, 12345678901234567.0});
  std::ofstream log(dir + "/ref_tns.txt");
  for (const char* name : {"ok.tns", "rank3.tns", "bad_rank.tns", "zero_based.tns", "short.tns", "empty.tns"}) {
    try {
      CooData t = read_tns(dir + "/" + name);
      log << name << " ok rank " << t.coords.size() << " extents";
      for (auto e : t.shape.extents) log << " " << e;
      log << " nnz " << t.values.size() << " :";
      for (size_t e = 0; e < t.values.size(); ++e) {
        log << " (";
        for (size_t k = 0; k < t.coords.size(); ++k) log << t.coords[k][e] << (k + 1 < t.coords.size() ? "," : "");
        log << ")=" << t.values[e];
      }
      log << "\n";
    } catch (const Error& e) {
      std::string msg = e.what();
      const size_t at = msg.find(name);  // strip the directory
      log << name << " error " << static_cast<int>(e.kind()) << " " << (at == std::string::npos ? msg : msg.substr(at))
          << "\n";
    }
  }
  return 0;
}
