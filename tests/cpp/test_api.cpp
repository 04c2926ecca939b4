// Drop-in check: reference-style code (the load_operand / cmd_kernel flow of
// cli.hpp:60-65, 222-263 and the reference test patterns) compiled against
// include/sparseforge_b200/sparseforge.hpp and run on the GPU. Expected
// values are the reference goldens for matrix A (proj/tests/oracle_data.hpp).
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "sparseforge_b200/sparseforge.hpp"

using namespace sparseforge;

static int failures = 0;
#define EXPECT(cond)                                                        \
  do {                                                                      \
    if (!(cond)) {                                                          \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);          \
      ++failures;                                                           \
    }                                                                       \
  } while (0)

template <class A, class B>
static bool same(const A& a, const B& b) {
  if (a.size() != b.size()) return false;
  for (size_t i = 0; i < a.size(); ++i)
    if (a[i] != b[i]) return false;
  return true;
}

int main(int argc, char** argv) {
  const std::vector<std::int64_t> coo_d0 = {0, 1, 2, 2, 2, 4}, coo_d1 = {0, 1, 1, 2, 3, 3};
  const std::vector<double> coo_val = {1, 2, 3, 4, 5, 6};
  // shuffled input (FromCooSortsInput, test_tensor.cpp:47-54)
  WorkingTensor t = from_coo(TensorShape{{5, 4}}, {{4, 0, 2, 2, 1, 2}, {3, 0, 3, 1, 1, 2}},
                             {6, 1, 5, 3, 2, 4});
  std::vector<std::vector<std::int64_t>> coords;
  std::vector<double> values;
  t.download(coords, values);
  EXPECT(same(coords[0], coo_d0) && same(coords[1], coo_d1) && same(values, coo_val));

  // plan goldens (oracle_data.hpp:151, test_planner.cpp:40-42)
  EXPECT(same(plan_lines(plan_conversion(resolve_format("COO"), resolve_format("CSR"))),
              std::vector<std::string>{"Fill(0)", "Merge(0)"}));

  // CSR through the reference's load_operand flow
  FormatEncoding csr = resolve_format("CSR");
  WorkingTensor a = t;
  convert_structure(a, resolve_format("map (d0, d1) -> (d0, d1); trim(0,1)"), csr);
  MaterializedTensor mat = materialize(a, infer_storage(csr));
  EXPECT(same(mat.levels[1].ptr, std::vector<std::int64_t>{0, 1, 2, 5, 5, 6}));
  EXPECT(same(mat.levels[1].idx, std::vector<std::int64_t>{0, 1, 1, 2, 3, 3}));
  EXPECT(same(mat.values, coo_val));
  EXPECT(explain_storage(infer_storage(csr)) == "L0: size | L1: ptr, idx | val");

  // spmv_y = A * 1 (oracle_data.hpp:125) for every covered format
  DenseTensor ones(TensorShape{{4}});
  for (auto& v : ones.data) v = 1.0;
  for (const char* name : {"COO", "CSR", "CSC", "DCSR", "ELL", "BCSR(2,2)", "BCSR(4,4)", "DOK", "LIL"}) {
    FormatEncoding enc = resolve_format(name);
    WorkingTensor w = t;
    convert_structure(w, resolve_format("COO"), enc);
    DenseTensor y = run_kernel(spmv_kernel(), {KernelOperand::from_materialized(enc, materialize(w, infer_storage(enc))),
                                               KernelOperand::from_dense(ones)});
    EXPECT(same(y.data, std::vector<double>{1, 2, 12, 0, 6}));
  }

  // LIL = CSR + pack(0,1) (formats.hpp:45): the CSR goldens (oracle_data.hpp:34-36)
  // with the AoS layout over levels 0..1 (operators.hpp:424-430)
  {
    FormatEncoding lil = resolve_format("map (d0, d1) -> (d0, d1); merge(0), trim(1,1), pack(0,1)");
    EXPECT(lil.name == "LIL");
    EXPECT(same(plan_lines(plan_conversion(resolve_format("COO"), lil)),
                std::vector<std::string>{"Fill(0)", "Merge(0)", "Pack(0,1)"}));
    WorkingTensor w = t;
    convert_structure(w, resolve_format("COO"), lil);
    MaterializedTensor m = materialize(w, infer_storage(lil));
    EXPECT(m.layout.kind == ValueLayoutKind::AoS && m.layout.aos_start == 0 && m.layout.aos_end == 1);
    EXPECT(same(m.levels[1].ptr, std::vector<std::int64_t>{0, 1, 2, 5, 5, 6}));
    EXPECT(same(m.levels[1].idx, std::vector<std::int64_t>{0, 1, 1, 2, 3, 3}));
    EXPECT(same(m.values, coo_val));
    EXPECT(explain_storage(infer_storage(lil)) == "L0: size | L1: ptr, idx | val | pack(0,1)");
  }

  // ELL and BCSR(2,2) goldens (oracle_data.hpp:67-97)
  {
    FormatEncoding ell = resolve_format("ELL");
    WorkingTensor w = t;
    convert_structure(w, resolve_format("COO"), ell);
    MaterializedTensor m = materialize(w, infer_storage(ell));
    EXPECT(same(m.levels[2].idx, std::vector<std::int64_t>{0, 1, 1, 0, 3, 0, 0, 2, 0, 0, 0, 0, 3, 0, 0}));
    EXPECT(same(m.values, std::vector<double>{1, 2, 3, 0, 6, 0, 0, 4, 0, 0, 0, 0, 5, 0, 0}));
    FormatEncoding b = resolve_format("BCSR(2,2)");
    WorkingTensor w2 = t;
    convert_structure(w2, resolve_format("COO"), b);
    MaterializedTensor mb = materialize(w2, infer_storage(b));
    EXPECT(same(mb.levels[1].ptr, std::vector<std::int64_t>{0, 1, 3, 4}));
    EXPECT(same(mb.levels[1].idx, std::vector<std::int64_t>{0, 0, 1, 1}));
    EXPECT(same(mb.values, std::vector<double>{1, 0, 0, 2, 0, 3, 0, 0, 4, 5, 0, 0, 0, 6, 0, 0}));
  }

  // SpMM: C = A B with B = [1, 10] per row
  {
    DenseTensor b(TensorShape{{4, 2}});
    for (int r = 0; r < 4; ++r) b.at({r, 0}) = 1, b.at({r, 1}) = 10;
    FormatEncoding enc = resolve_format("CSR");
    WorkingTensor w = t;
    convert_structure(w, resolve_format("COO"), enc);
    DenseTensor c = run_kernel(spmm_kernel(), {KernelOperand::from_materialized(enc, materialize(w, infer_storage(enc))),
                                               KernelOperand::from_dense(b)});
    EXPECT(same(c.data, std::vector<double>{1, 10, 2, 20, 12, 120, 0, 0, 6, 60}));
  }

  // decompose (row_nnz = 1 1 3 0 1, oracle_data.hpp:107)
  {
    DecomposeRule rule;
    rule.min_sum = 2;
    DecomposeResult r = decompose(t, rule);
    EXPECT(r.totals.at({2}) == 3 && r.totals.at({3}) == 0);
    EXPECT(r.selected.entry_count() == 3 && r.remainder.entry_count() == 3);
  }

  // errors keep the reference ErrorKind (tensor.hpp:131-153)
  try {
    from_coo(TensorShape{{3, 3}}, {{1, 1}, {2, 2}}, {5.0, 7.0});
    EXPECT(false);
  } catch (const Error& e) {
    EXPECT(e.kind() == ErrorKind::DuplicateCoordinate);
  }
  try {
    from_coo(TensorShape{{3, 3}}, {{3}, {0}}, {1.0});
    EXPECT(false);
  } catch (const Error& e) {
    EXPECT(e.kind() == ErrorKind::InvalidOperation);
  }
  try {
    resolve_format("NOPE");
    EXPECT(false);
  } catch (const Error& e) {
    EXPECT(e.kind() == ErrorKind::Parse);
  }
  WorkingTensor s = from_coo(TensorShape{{3, 3}}, {{1, 0, 1}, {2, 0, 2}}, {5.0, 1.0, 7.0}, true);
  s.download(coords, values);
  EXPECT(same(values, std::vector<double>{1.0, 12.0}));

  if (argc > 1) {  // Matrix Market ingest (io.hpp:50): tests/golden/mm fixtures
    const std::string dir = argv[1];
    CooData d = read_matrix_market(dir + "/real_symmetric.mtx");
    EXPECT(d.shape.extents == (std::vector<std::int64_t>{4, 4}));
    EXPECT(same(d.coords[0], std::vector<std::int64_t>{0, 0, 1, 1, 2, 2, 3, 3}));
    EXPECT(same(d.coords[1], std::vector<std::int64_t>{0, 1, 0, 2, 1, 3, 2, 3}));
    EXPECT(same(d.values, std::vector<double>{2, -1, -1, -1, -1, -1, -1, 2}));
    WorkingTensor w = load_matrix_market(dir + "/pattern_symmetric.mtx");
    w.download(coords, values);
    EXPECT(values.size() == 6);
    try {
      read_matrix_market(dir + "/err_missing_value.mtx");
      EXPECT(false);
    } catch (const Error& e) {
      EXPECT(e.kind() == ErrorKind::Parse);
      EXPECT(std::string(e.what()).find(":4: missing value") != std::string::npos);
    }
  }
  {  // USPT container round trip (io.hpp:240, 283)
    WorkingTensor a = from_coo(TensorShape{{5, 4}}, {coo_d0, coo_d1}, coo_val);
    convert_structure(a, resolve_format("COO"), resolve_format("CSR"));
    MaterializedTensor ma = materialize(a, infer_storage(resolve_format("CSR")));
    write_container("/tmp/sfg_test_api.uspt", ma);
    MaterializedTensor mb = read_container("/tmp/sfg_test_api.uspt");
    EXPECT(mb.levels.size() == 2 && same(mb.levels[1].ptr, ma.levels[1].ptr) &&
           same(mb.levels[1].idx, ma.levels[1].idx) && same(mb.values, ma.values));
  }
  {  // two sparse operands (kernel.hpp:424): A (5x4) times A^T-shaped B (4x5)
    WorkingTensor a = from_coo(TensorShape{{5, 4}}, {coo_d0, coo_d1}, coo_val);
    WorkingTensor b = from_coo(TensorShape{{4, 5}}, {coo_d1, coo_d0}, coo_val);
    convert_structure(a, resolve_format("COO"), resolve_format("CSR"));
    MaterializedTensor ma = materialize(a, infer_storage(resolve_format("CSR")));
    MaterializedTensor mb = materialize(b, infer_storage(resolve_format("COO")));
    DenseTensor c = run_kernel(spgemm_kernel(), {KernelOperand::from_materialized(ma.enc, ma),
                                                 KernelOperand::from_materialized(mb.enc, mb)});
    // (A A^T)[2][2] = 3*3 + 4*4 + 5*5 = 50; [0][0] = 1; [2][4] = 5*6 = 30
    EXPECT(c.data[2 * 5 + 2] == 50 && c.data[0] == 1 && c.data[2 * 5 + 4] == 30);
  }
  {  // row-partitioned path, one rank: chunk 0 = the plain product
    WorkingTensor a = from_coo(TensorShape{{5, 4}}, {coo_d0, coo_d1}, coo_val);
    convert_structure(a, resolve_format("COO"), resolve_format("CSR"));
    MaterializedTensor ma = materialize(a, infer_storage(resolve_format("CSR")));
    DenseTensor x(TensorShape{{4}});
    for (auto& v : x.data) v = 1.0;
    b200::Comm comm(1, 0, b200::comm_unique_id());
    DenseTensor y = run_kernel_rowpart(spmv_kernel(), {KernelOperand::from_materialized(ma.enc, ma),
                                                       KernelOperand::from_dense(x)}, comm, 7);
    const std::vector<double> want{1, 2, 12, 0, 6};  // spmv_y (oracle_data.hpp:125)
    EXPECT(y.data.size() == 7);
    for (size_t i = 0; i < want.size(); ++i) EXPECT(y.data[i] == want[i]);
  }
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}
