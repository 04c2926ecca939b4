// ref_shim.cpp — CPU ORACLE (test infrastructure only).
//
// A C-ABI around the UNMODIFIED reference headers (sparse-forge,
// /root/reference/proj/include). Built by oracle/Makefile into
// oracle/_ref/libsfref.so with -I pointing at the reference tree; no
// reference source is copied into this repository. The accessor surface
// mirrors oracle/sfo.h so tests can run the same checks against the real
// reference (sfr_*) and the C restatement (sfo_*).
//
// Call chain per entry point (reference file:line):
//   sfr_from_coo       -> from_coo                    tensor.hpp:118
//   sfr_convert        -> resolve_format               formats.hpp:92
//                         convert_structure(COO->dst)  planner.hpp:261
//                         materialize(infer_storage)   storage.hpp:97, 35
//   sfr_spmv/sfr_spmm  -> KernelOperand::from_materialized + run_kernel
//                                                      kernel.hpp:80, 236
//   sfr_decompose_rows -> decompose(count rule)        decompose.hpp:30
//   sfr_plan           -> plan_conversion + plan_lines planner.hpp:95, 22
//   sfr_read_mm        -> read_matrix_market + from_coo io.hpp:50-121
//   sfr_convert_from   -> convert_structure from a non-COO structure
//   sfr_spgemm         -> run_kernel(spgemm_kernel(), {A, B})   kernel.hpp:424
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "sparseforge/decompose.hpp"
#include "sparseforge/formats.hpp"
#include "sparseforge/io.hpp"
#include "sparseforge/kernel.hpp"
#include "sparseforge/parse.hpp"
#include "sparseforge/planner.hpp"
#include "sparseforge/storage.hpp"
#include "sparseforge/tensor.hpp"

using namespace sparseforge;

namespace {

thread_local std::string g_err;

struct RefCoo {
  WorkingTensor t;
};

struct RefMat {
  FormatEncoding enc;
  MaterializedTensor m;
};

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return 1 + static_cast<int>(e.kind());
  } catch (const std::exception& e) {
    g_err = e.what();
    return 100;
  }
}

int copy_text(const std::string& s, char* buf, int64_t len) {
  if (len <= 0) return 0;
  size_t n = std::min<size_t>(s.size(), static_cast<size_t>(len - 1));
  std::memcpy(buf, s.data(), n);
  buf[n] = 0;
  return 0;
}

}  // namespace

extern "C" {

const char* sfr_last_error() { return g_err.c_str(); }

int sfr_from_coo(int64_t m, int64_t n, int64_t nnz, const int64_t* row, const int64_t* col,
                 const double* val, int sum_duplicates, void** out) {
  *out = nullptr;
  return guard([&] {
    std::vector<std::vector<int64_t>> coords = {std::vector<int64_t>(row, row + nnz),
                                                std::vector<int64_t>(col, col + nnz)};
    std::vector<double> values(val, val + nnz);
    auto* c = new RefCoo{from_coo(TensorShape{{m, n}}, coords, values, sum_duplicates != 0)};
    *out = c;
  });
}

int64_t sfr_coo_nnz(void* h) { return static_cast<int64_t>(static_cast<RefCoo*>(h)->t.entry_count()); }

int sfr_coo_get(void* h, int64_t* row, int64_t* col, double* val) {
  const WorkingTensor& t = static_cast<RefCoo*>(h)->t;
  size_t n = t.entry_count();
  if (row) std::memcpy(row, t.coords[0].data(), n * sizeof(int64_t));
  if (col) std::memcpy(col, t.coords[1].data(), n * sizeof(int64_t));
  if (val) std::memcpy(val, t.values.data(), n * sizeof(double));
  return 0;
}

void sfr_coo_free(void* h) { delete static_cast<RefCoo*>(h); }

// Matrix Market file -> canonical COO, exactly as the reference CLI loads a
// COO operand: read_matrix_market, then from_coo (io.hpp:50, tensor.hpp:118).
int sfr_read_mm(const char* path, int sum_duplicates, void** out) {
  *out = nullptr;
  return guard([&] {
    CooData d = read_matrix_market(path);
    *out = new RefCoo{from_coo(d.shape, d.coords, d.values, sum_duplicates != 0)};
  });
}

// write_container of the reference's materialized `fmt` form of a COO.
int sfr_write_container(void* h, const char* fmt, const char* path) {
  return guard([&] {
    WorkingTensor t = static_cast<RefCoo*>(h)->t;
    FormatEncoding dst = resolve_format(fmt);
    convert_structure(t, resolve_format("COO"), dst);
    write_container(path, materialize(t, infer_storage(dst)));
  });
}

int sfr_coo_shape(void* h, int64_t* m, int64_t* n) {
  const WorkingTensor& t = static_cast<RefCoo*>(h)->t;
  *m = t.shape.extents[0];
  *n = t.shape.extents[1];
  return 0;
}

int sfr_convert(void* h, const char* fmt, void** out) {
  *out = nullptr;
  return guard([&] {
    WorkingTensor t = static_cast<RefCoo*>(h)->t;
    FormatEncoding dst = resolve_format(fmt);
    convert_structure(t, resolve_format("COO"), dst);
    auto* m = new RefMat{dst, materialize(t, infer_storage(dst))};
    *out = m;
  });
}

// A tensor held in structure `mid` converted to `dst` (convert_structure
// from a non-COO source, planner.hpp:95-252: normalize, realign, regrow).
int sfr_convert_from(void* h, const char* mid, const char* fmt, void** out) {
  *out = nullptr;
  return guard([&] {
    WorkingTensor t = static_cast<RefCoo*>(h)->t;
    FormatEncoding src = resolve_format(mid), dst = resolve_format(fmt);
    convert_structure(t, resolve_format("COO"), src);
    convert_structure(t, src, dst);
    *out = new RefMat{dst, materialize(t, infer_storage(dst))};
  });
}

int sfr_mat_nlevels(void* h) { return static_cast<int>(static_cast<RefMat*>(h)->m.levels.size()); }

int sfr_mat_level_info(void* h, int l, int64_t info[6]) {
  const MaterializedLevel& lev = static_cast<RefMat*>(h)->m.levels.at(static_cast<size_t>(l));
  info[0] = (lev.storage.size ? 1 : 0) | (lev.storage.ptr ? 2 : 0) | (lev.storage.idx ? 4 : 0) |
            (lev.storage.dense_vector ? 8 : 0);
  info[1] = lev.bounds.lo;
  info[2] = lev.bounds.hi;
  info[3] = static_cast<int64_t>(lev.node_count);
  info[4] = static_cast<int64_t>(lev.idx.size());
  info[5] = static_cast<int64_t>(lev.ptr.size());
  return 0;
}

int sfr_mat_level_idx(void* h, int l, int64_t* out) {
  const auto& v = static_cast<RefMat*>(h)->m.levels.at(static_cast<size_t>(l)).idx;
  if (!v.empty()) std::memcpy(out, v.data(), v.size() * sizeof(int64_t));
  return 0;
}

int sfr_mat_level_ptr(void* h, int l, int64_t* out) {
  const auto& v = static_cast<RefMat*>(h)->m.levels.at(static_cast<size_t>(l)).ptr;
  if (!v.empty()) std::memcpy(out, v.data(), v.size() * sizeof(int64_t));
  return 0;
}

int64_t sfr_mat_nvals(void* h) { return static_cast<int64_t>(static_cast<RefMat*>(h)->m.values.size()); }

int sfr_mat_values(void* h, double* out) {
  const auto& v = static_cast<RefMat*>(h)->m.values;
  if (!v.empty()) std::memcpy(out, v.data(), v.size() * sizeof(double));
  return 0;
}

// ValueLayout of the materialized tensor (tensor.hpp:58-64; set by Pack,
// storage.hpp:128-133): {0 SoA / 1 AoS, aos_start, aos_end}.
int sfr_mat_layout(void* h, int64_t out[3]) {
  const auto& l = static_cast<RefMat*>(h)->m.layout;
  out[0] = l.kind == ValueLayoutKind::AoS ? 1 : 0;
  out[1] = static_cast<int64_t>(l.aos_start);
  out[2] = static_cast<int64_t>(l.aos_end);
  return 0;
}

// Partition value ranges (storage.hpp:220-231), as (begin, end) pairs.
int64_t sfr_mat_npartitions(void* h) { return static_cast<int64_t>(static_cast<RefMat*>(h)->m.partitions.size()); }
int sfr_mat_partitions(void* h, int64_t* out) {
  const auto& p = static_cast<RefMat*>(h)->m.partitions;
  for (size_t i = 0; i < p.size(); ++i) {
    out[2 * i] = static_cast<int64_t>(p[i].first);
    out[2 * i + 1] = static_cast<int64_t>(p[i].second);
  }
  return 0;
}

void sfr_mat_free(void* h) { delete static_cast<RefMat*>(h); }

int sfr_spmv(void* h, const double* x, double* y, int threads) {
  return guard([&] {
    RefMat* a = static_cast<RefMat*>(h);
    int64_t m = a->m.logical_shape.extents[0], n = a->m.logical_shape.extents[1];
    DenseTensor xd(TensorShape{{n}});
    std::memcpy(xd.data.data(), x, static_cast<size_t>(n) * sizeof(double));
    KernelOptions opt;
    opt.threads = threads;
    DenseTensor y_out = run_kernel(
        spmv_kernel(), {KernelOperand::from_materialized(a->enc, a->m), KernelOperand::from_dense(xd)},
        opt);
    std::memcpy(y, y_out.data.data(), static_cast<size_t>(m) * sizeof(double));
  });
}

int sfr_spmm(void* h, const double* b, int64_t nd, double* c, int threads) {
  return guard([&] {
    RefMat* a = static_cast<RefMat*>(h);
    int64_t m = a->m.logical_shape.extents[0], n = a->m.logical_shape.extents[1];
    DenseTensor bd(TensorShape{{n, nd}});
    std::memcpy(bd.data.data(), b, static_cast<size_t>(n * nd) * sizeof(double));
    KernelOptions opt;
    opt.threads = threads;
    DenseTensor c_out = run_kernel(
        spmm_kernel(), {KernelOperand::from_materialized(a->enc, a->m), KernelOperand::from_dense(bd)},
        opt);
    std::memcpy(c, c_out.data.data(), static_cast<size_t>(m * nd) * sizeof(double));
  });
}

// run_kernel(spgemm_kernel(), {A, B}) with two sparse operands
// (kernel.hpp:53, 424-567): dense C[M x N2] (f64).
int sfr_spgemm(void* ha, void* hb, double* c, char* mode, int64_t mode_len) {
  return guard([&] {
    RefMat* a = static_cast<RefMat*>(ha);
    RefMat* b = static_cast<RefMat*>(hb);
    IterationPlan plan;
    DenseTensor c_out = run_kernel(spgemm_kernel(),
                                   {KernelOperand::from_materialized(a->enc, a->m),
                                    KernelOperand::from_materialized(b->enc, b->m)},
                                   KernelOptions{}, &plan);
    std::memcpy(c, c_out.data.data(), c_out.data.size() * sizeof(double));
    if (mode) copy_text(plan.gemm_mode, mode, mode_len);
  });
}

int sfr_decompose_rows(void* h, int64_t min_sum, void** sel, void** rem, int64_t* totals) {
  *sel = *rem = nullptr;
  return guard([&] {
    const WorkingTensor& t = static_cast<RefCoo*>(h)->t;
    DecomposeRule rule;
    rule.query = parse_query(
        "sum(value) groupBy (d0, d1) -> (d0) with value ne 0 -> 1 | otherwise -> 0");
    rule.min_sum = min_sum;
    DecomposeResult r = decompose(t, rule);
    if (totals)
      for (const auto& [k, v] : r.totals) totals[k.at(0)] = v;
    *sel = new RefCoo{std::move(r.selected)};
    *rem = new RefCoo{std::move(r.remainder)};
  });
}

// decompose by r x c blocks with the block count rule (decompose.hpp:30-63)
int sfr_decompose_blocks(void* h, int64_t r, int64_t c, int64_t min_sum, void** sel, void** rem) {
  *sel = *rem = nullptr;
  return guard([&] {
    const WorkingTensor& t = static_cast<RefCoo*>(h)->t;
    DecomposeRule rule;
    rule.query = parse_query("sum(value) groupBy (d0, d1) -> (d0/" + std::to_string(r) + ", d1/" + std::to_string(c) +
                             ") with value ne 0 -> 1 | otherwise -> 0");
    rule.min_sum = min_sum;
    DecomposeResult d = decompose(t, rule);
    *sel = new RefCoo{std::move(d.selected)};
    *rem = new RefCoo{std::move(d.remainder)};
  });
}

int sfr_plan(const char* src, const char* dst, char* buf, int64_t len) {
  return guard([&] {
    std::string out;
    for (const auto& line : plan_lines(plan_conversion(resolve_format(src), resolve_format(dst))))
      out += line + "\n";
    copy_text(out, buf, len);
  });
}

int sfr_storage_explain(const char* fmt, char* buf, int64_t len) {
  return guard([&] { copy_text(explain_storage(infer_storage(resolve_format(fmt))), buf, len); });
}

}  // extern "C"
