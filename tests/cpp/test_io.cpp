// io.hpp / tensor.hpp utilities of the drop-in C++ API: the host-side text
// formats against the reference's own outputs (tests/golden/io, made by
// gen_io.cpp against the unmodified headers), and — with --gpu — the
// device round trips from_dense -> convert -> to_dense / to_coo_data /
// materialize -> dematerialize.
#include <cmath>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <sstream>

#include "sparseforge_b200/sparseforge.hpp"

using namespace sparseforge;

static std::string slurp(const std::string& p) {
  std::ifstream in(p);
  std::stringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

#define CHECK(c)                                                      \
  do {                                                                \
    if (!(c)) {                                                       \
      std::cerr << "FAIL " << __LINE__ << ": " #c << std::endl;       \
      return 1;                                                       \
    }                                                                 \
  } while (0)

int main(int argc, char** argv) {
  const std::string dir = argv[1], tmp = argv[2];
  const bool gpu = argc > 3 && std::string(argv[3]) == "--gpu";
  CooData d;
  d.shape.extents = {4, 5};
  d.coords = {{0, 1, 3, 3, 2}, {4, 0, 2, 3, 1}};
  d.values = {0.1, -2.5, 1.0 / 3.0, 6.02214076e23, 1e-300};
  write_matrix_market(tmp + "/out.mtx", d);
  CHECK(slurp(tmp + "/out.mtx") == slurp(dir + "/ref_out.mtx"));
  write_vector_text(tmp + "/vec.txt", {0.1, -0.0, 3.0, 1.0 / 7.0, 12345678901234567.0});
  CHECK(slurp(tmp + "/vec.txt") == slurp(dir + "/ref_vec.txt"));
  const std::vector<double> back = read_vector_text(tmp + "/vec.txt");
  CHECK(back.size() == 5 && back[0] == 0.1 && back[3] == 1.0 / 7.0);
  std::ostringstream log;
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
      const size_t at = msg.find(name);
      log << name << " error " << static_cast<int>(e.kind()) << " " << (at == std::string::npos ? msg : msg.substr(at))
          << "\n";
    }
  }
  CHECK(log.str() == slurp(dir + "/ref_tns.txt"));
  try {
    write_matrix_market("/nonexistent-dir/x.mtx", d);
    CHECK(false);
  } catch (const Error& e) {
    CHECK(e.kind() == ErrorKind::Io);
  }
  if (gpu) {
    DenseTensor a(TensorShape{{5, 7}});
    a.at({0, 1}) = 2.0;
    a.at({2, 6}) = -1.5;
    a.at({4, 0}) = 0.25;
    a.at({4, 6}) = 8.0;
    WorkingTensor w = from_dense(a);
    CHECK(equal_dense(to_dense(w), a));
    convert_structure(w, resolve_format("COO"), resolve_format("CSR"));
    CHECK(equal_dense(to_dense(w), a));
    CooData c = to_coo_data(w);
    CHECK(c.values.size() == 4 && c.coords[0][1] == 2 && c.coords[1][1] == 6 && c.values[3] == 8.0);
    FormatEncoding enc = resolve_format("CSR");
    MaterializedTensor m = materialize(w, infer_storage(enc));
    WorkingTensor w2 = dematerialize(m, enc);
    CHECK(equal_dense(to_dense(w2), a));
    try {
      dematerialize(m, resolve_format("ELL"));
      CHECK(false);
    } catch (const Error& e) {
      CHECK(e.kind() == ErrorKind::InvalidOperation);
    }
  }
  std::cout << "OK" << std::endl;
  return 0;
}
