// convert_src.cu — conversions from compressed sources (SURVEY.md §8f
// rank 2): CSR, DCSR, CSC and BCSR tensors back to a canonical COO
// (dematerialize, storage.hpp:284-343), then on to any target through the
// COO conversions.
//
// Reference semantics (planner.hpp:95-252, operators.hpp:302-345): a source
// whose index map equals the target's only adjusts level flags; otherwise
// the source is first normalized — split, and every untrimmed level l
// trimmed. Trim(l) groups the entries by their path through level l and
// drops every group whose values are all zero. So, measured against the
// reference (tests/test_gpu_convert_src.py):
//   CSR  (Fill(0)): Trim(0) unless the target is CSR — rows whose stored
//        values are all zero disappear;
//   DCSR: nothing is trimmed;
//   CSC  (Fill(0) over columns): Trim(0) unless the target is CSC —
//        all-zero columns disappear;
//   BCSR (Fill(3), Fill(2), Fill(0), Vectorize): every zero value
//        disappears (block padding included), and the extents stay those of
//        the whole block grid (TileUnion(0, r): ceil(M/r) r x ceil(N/c) c);
//   ELL (an indirect level): UnsupportedSource.
// The same format and parameters on both sides is the identity (a copy).
#include <cuda_bf16.h>

#include <algorithm>

#include "devutil.cuh"
#include "internal.cuh"

namespace sfg {

namespace {

constexpr int kBlock = 256;
constexpr int kCompactItems = 16;
constexpr int kCompactTile = kBlock * kCompactItems;

// Row ids of a row-compressed level: warp per row (rows may be long).
// rows == nullptr: row p is p (CSR); otherwise rows[p] (DCSR).
__global__ void __launch_bounds__(kBlock) k_expand_rows(const int32_t* __restrict__ ptr,
                                                         const int32_t* __restrict__ rows, int64_t nrows,
                                                         int32_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < nrows; p += warps) {
    const int32_t s = __ldg(ptr + p), e = __ldg(ptr + p + 1);
    const int32_t r = rows ? __ldg(rows + p) : (int32_t)p;
    for (int32_t k = s + lane; k < e; k += 32) out[k] = r;
  }
}

// keep[p] = row p holds a nonzero value (Trim(0) over a row-compressed level).
__global__ void __launch_bounds__(kBlock) k_row_nonzero(const int32_t* __restrict__ ptr,
                                                         const float* __restrict__ val, int64_t nrows,
                                                         uint8_t* __restrict__ keep) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < nrows; p += warps) {
    const int32_t s = __ldg(ptr + p), e = __ldg(ptr + p + 1);
    bool nz = false;
    for (int32_t k = s + lane; k < e && !nz; k += 32) nz = __ldg(val + k) != 0.f;
    nz = __any_sync(kFull, nz);
    if (lane == 0) keep[p] = nz;
  }
}

// Order-preserving compaction of (row, col, val) entries: an entry stays when
// keep_row[row] (row trim) or, with keep_row == nullptr, when its value is
// nonzero (leaf trim). Single-pass look-back scan.
__global__ void __launch_bounds__(kBlock) k_compact(const int32_t* __restrict__ row, const int32_t* __restrict__ col,
                                                     const float* __restrict__ val, int64_t n,
                                                     const uint8_t* __restrict__ keep_row,
                                                     int32_t* __restrict__ orow, int32_t* __restrict__ ocol,
                                                     float* __restrict__ oval, unsigned long long* __restrict__ status,
                                                     uint32_t epoch, int32_t* __restrict__ total_out) {
  __shared__ uint32_t smem[34];
  __shared__ uint32_t slot;
  const int64_t e0 = (int64_t)blockIdx.x * kCompactTile + (int64_t)threadIdx.x * kCompactItems;
  uint32_t mask = 0;
#pragma unroll
  for (int i = 0; i < kCompactItems; ++i) {
    const int64_t e = e0 + i;
    if (e < n && (keep_row ? keep_row[row[e]] != 0 : val[e] != 0.f)) mask |= 1u << i;
  }
  uint32_t total;
  const uint32_t excl = block_exclusive_scan<uint32_t, kBlock>(__popc(mask), smem, &total);
  uint32_t pos = lookback_prefix(status, epoch, blockIdx.x, total, &slot) + excl;
  while (mask) {
    const int i = __ffs(mask) - 1;
    mask &= mask - 1;
    orow[pos] = row[e0 + i];
    ocol[pos] = col[e0 + i];
    oval[pos] = val[e0 + i];
    ++pos;
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == blockDim.x - 1) *total_out = (int32_t)(pos);
}

// BCSR slots -> (row, col, val) of the nonzero ones, in storage order
// (block-major, row-major inside a block); the caller sorts.
template <typename T>
__global__ void __launch_bounds__(kBlock) k_bcsr_slots(const int32_t* __restrict__ bptr,
                                                        const int32_t* __restrict__ bcol, const T* __restrict__ bval,
                                                        int64_t nbr, int32_t r, int32_t c, int32_t rb, int32_t cb,
                                                        int32_t* __restrict__ orow, int32_t* __restrict__ ocol,
                                                        float* __restrict__ oval,
                                                        unsigned long long* __restrict__ count) {
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int lane = threadIdx.x & 31;
  const int bs = rb * cb;
  for (int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < nbr; b += warps) {
    const int32_t s = __ldg(bptr + b), e = __ldg(bptr + b + 1);
    for (int32_t k = s; k < e; ++k) {
      const int32_t c0 = __ldg(bcol + k) * c;
      for (int q = lane; q < bs; q += 32) {
        const float v = (float)bval[(int64_t)k * bs + q];
        const bool nz = v != 0.f;
        const unsigned m = __ballot_sync(__activemask(), nz);
        unsigned long long base = 0;
        const int leader = __ffs(__activemask()) - 1;
        if (lane == leader && m) base = atomicAdd(count, (unsigned long long)__popc(m));
        base = __shfl_sync(__activemask(), base, leader);
        if (nz) {
          const unsigned long long at = base + __popc(m & ((1u << lane) - 1u));
          orow[at] = (int32_t)(b * r + q / cb);
          ocol[at] = c0 + q % cb;
          oval[at] = v;
        }
      }
    }
  }
}

// ELL slots holding a nonzero value, as unordered (row, col, val) triples:
// the padding cells (column 0, value 0) and explicit zeros drop out — a zero
// slot contributes 0 * B[col] to a product, which is what the reference's
// walk over every slot adds (kernel.hpp:147-153).
__global__ void __launch_bounds__(kBlock) k_ell_nonzeros(const int32_t* __restrict__ idx,
                                                         const float* __restrict__ val, int64_t m, int64_t k,
                                                         int32_t* __restrict__ orow, int32_t* __restrict__ ocol,
                                                         float* __restrict__ oval,
                                                         unsigned long long* __restrict__ count) {
  const int lane = threadIdx.x & 31;
  for (int64_t cell = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; cell - lane < k * m;
       cell += (int64_t)gridDim.x * blockDim.x) {
    const bool in = cell < k * m;
    const float v = in ? __ldg(val + cell) : 0.f;
    const bool nz = in && v != 0.f;
    const unsigned msk = __ballot_sync(kFull, nz);
    unsigned long long base = 0;
    if (lane == 0 && msk) base = atomicAdd(count, (unsigned long long)__popc(msk));
    base = __shfl_sync(kFull, base, 0);
    if (nz) {
      const unsigned long long at = base + __popc(msk & ((1u << lane) - 1u));
      orow[at] = (int32_t)(cell % m);
      ocol[at] = __ldg(idx + cell);
      oval[at] = v;
    }
  }
}

// BELL values that are nonzero, as unordered (row, col, val) triples
// (padding cells and the zero fill of blocks drop out).
__global__ void __launch_bounds__(kBlock) k_bell_nonzeros(const int32_t* __restrict__ bcol,
                                                          const float* __restrict__ val, int64_t nbr, int64_t cells,
                                                          int32_t b, int32_t rb, int32_t cb,
                                                          int32_t* __restrict__ orow, int32_t* __restrict__ ocol,
                                                          float* __restrict__ oval,
                                                          unsigned long long* __restrict__ count) {
  const int lane = threadIdx.x & 31;
  const int bs = rb * cb;
  const int64_t total = cells * bs;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e - lane < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const bool in = e < total;
    const float v = in ? __ldg(val + e) : 0.f;
    const bool nz = in && v != 0.f;
    const unsigned msk = __ballot_sync(kFull, nz);
    unsigned long long base = 0;
    if (lane == 0 && msk) base = atomicAdd(count, (unsigned long long)__popc(msk));
    base = __shfl_sync(kFull, base, 0);
    if (nz) {
      const int64_t cell = e / bs;
      const int q = (int)(e - cell * bs);
      const unsigned long long at = base + __popc(msk & ((1u << lane) - 1u));
      orow[at] = (int32_t)((cell % nbr) * b + q / cb);
      ocol[at] = __ldg(bcol + cell) * b + q % cb;
      oval[at] = v;
    }
  }
}

sfg_tensor* make_coo(sfg_context* ctx, int64_t m, int64_t n, int64_t nnz) {
  sfg_tensor* t = new_tensor(ctx, SFG_COO, m, n);
  t->nnz = nnz;
  t->row = dalloc_n<int32_t>(ctx, nnz);
  t->idx = dalloc_n<int32_t>(ctx, nnz);
  t->val = dalloc_n<float>(ctx, nnz);
  return t;
}

// Row-trimmed copy of a canonical COO whose rows are described by keep[].
sfg_tensor* compact(sfg_context* ctx, sfg_tensor* coo, const uint8_t* keep) {
  sfg_tensor* out = make_coo(ctx, coo->m, coo->n, coo->nnz);
  if (coo->nnz) {
    const int tiles = (int)ceil_div(coo->nnz, kCompactTile);
    auto* tot = static_cast<int32_t*>(scratch(ctx, 64));
    SFG_LAUNCH(k_compact, tiles, kBlock, 0, ctx->stream, coo->row, coo->idx, static_cast<const float*>(coo->val),
               coo->nnz, keep, out->row, out->idx, static_cast<float*>(out->val), lookback_status(ctx, tiles),
               ctx->epoch++, tot);
    int32_t kept = 0;
    read_back(ctx, tot, 4, &kept);
    out->nnz = kept;
  }
  return out;
}

void free_tensor(sfg_tensor* t) {
  if (!t) return;
  free_tensor_arrays(t);
  delete t;
}

// Row-compressed (CSR / DCSR / CSC-as-CSR-of-the-transpose) -> canonical COO,
// optionally dropping the rows whose values are all zero.
sfg_tensor* row_compressed_to_coo(sfg_context* ctx, const int32_t* ptr, const int32_t* rows, int64_t nrows,
                                  const int32_t* idx, const float* val, int64_t nnz, int64_t m, int64_t n,
                                  bool trim_rows) {
  if (rows && trim_rows) raise(SFG_ERR_INVALID_OPERATION, "row trim expects a CSR-shaped level");
  sfg_tensor* coo = make_coo(ctx, m, n, nnz);
  if (nnz) {
    const int grid = (int)std::min<int64_t>(ceil_div(nrows, kBlock / 32), (int64_t)ctx->sms * 16);
    SFG_LAUNCH(k_expand_rows, grid, kBlock, 0, ctx->stream, ptr, rows, nrows, coo->row);
    SFG_CUDA(cudaMemcpyAsync(coo->idx, idx, nnz * 4, cudaMemcpyDeviceToDevice, ctx->stream));
    SFG_CUDA(cudaMemcpyAsync(coo->val, val, nnz * 4, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  if (!trim_rows || nnz == 0) return coo;
  // keep[] is indexed by the row coordinate (rows == nullptr: p is the row)
  uint8_t* keep = static_cast<uint8_t*>(dalloc(ctx, std::max<int64_t>(m, 1)));
  SFG_CUDA(cudaMemsetAsync(keep, 0, std::max<int64_t>(m, 1), ctx->stream));
  const int grid = (int)std::min<int64_t>(ceil_div(nrows, kBlock / 32), (int64_t)ctx->sms * 16);
  SFG_LAUNCH(k_row_nonzero, grid, kBlock, 0, ctx->stream, ptr, val, nrows, keep);
  sfg_tensor* out = compact(ctx, coo, keep);
  dfree(ctx, keep);
  free_tensor(coo);
  return out;
}

sfg_tensor* csc_to_coo(sfg_context* ctx, const sfg_tensor* s, bool trim_cols) {
  // The CSC of A is the CSR of A^T: expand it to the canonical COO of A^T
  // (all-zero columns of A = all-zero rows of A^T, trimmed there), let the
  // COO -> CSC conversion of A^T produce the CSR of A, expand that.
  sfg_tensor* at = row_compressed_to_coo(ctx, s->ptr, nullptr, s->n, s->idx, static_cast<const float*>(s->val),
                                         s->nnz, s->n, s->m, trim_cols);
  sfg_tensor* a_csr = nullptr;
  try {
    a_csr = coo_to_csc(ctx, at);  // column-compressed A^T == row-compressed A
  } catch (...) {
    free_tensor(at);
    throw;
  }
  free_tensor(at);
  sfg_tensor* out = nullptr;
  try {
    out = row_compressed_to_coo(ctx, a_csr->ptr, nullptr, s->m, a_csr->idx, static_cast<const float*>(a_csr->val),
                                a_csr->nnz, s->m, s->n, false);
  } catch (...) {
    free_tensor(a_csr);
    throw;
  }
  free_tensor(a_csr);
  return out;
}

sfg_tensor* bcsr_to_coo(sfg_context* ctx, const sfg_tensor* s) {
  // every zero disappears (Trim(3), Trim(2), Trim(0)); extents = the grid
  const int64_t m = s->nbr * s->br, n = s->nbc * s->bc;
  const int64_t slots = s->nnz * s->rb * s->cb;
  sfg_tensor* tmp = make_coo(ctx, m, n, slots);
  auto* count = static_cast<unsigned long long*>(scratch(ctx, 64));
  SFG_CUDA(cudaMemsetAsync(count, 0, 8, ctx->stream));
  const int grid = (int)std::min<int64_t>(ceil_div(s->nbr, kBlock / 32), (int64_t)ctx->sms * 16);
  if (s->nbr > 0) {
    if (s->dtype == SFG_BF16)
      SFG_LAUNCH(k_bcsr_slots<__nv_bfloat16>, grid, kBlock, 0, ctx->stream, s->ptr, s->idx,
                 static_cast<const __nv_bfloat16*>(s->val), s->nbr, (int32_t)s->br, (int32_t)s->bc, (int32_t)s->rb,
                 (int32_t)s->cb, tmp->row, tmp->idx, static_cast<float*>(tmp->val), count);
    else
      SFG_LAUNCH(k_bcsr_slots<float>, grid, kBlock, 0, ctx->stream, s->ptr, s->idx, static_cast<const float*>(s->val),
                 s->nbr, (int32_t)s->br, (int32_t)s->bc, (int32_t)s->rb, (int32_t)s->cb, tmp->row, tmp->idx,
                 static_cast<float*>(tmp->val), count);
  }
  unsigned long long nz = 0;
  read_back(ctx, count, 8, &nz);
  sfg_tensor* out = nullptr;
  try {
    out = sort_coo(ctx, m, n, (int64_t)nz, tmp->row, tmp->idx, static_cast<const float*>(tmp->val), false);
  } catch (...) {
    free_tensor(tmp);
    throw;
  }
  free_tensor(tmp);
  return out;
}

}  // namespace

// DCSC: as the CSC above, with the nonempty-column list as the A^T row ids
// (Split(0) Swap(0,1) Sort: no column trim — empty columns are already gone)
sfg_tensor* dcsc_to_coo(sfg_context* ctx, const sfg_tensor* s) {
  sfg_tensor* at = row_compressed_to_coo(ctx, s->ptr, s->row, tensor_nnr(s), s->idx,
                                         static_cast<const float*>(s->val), s->nnz, s->n, s->m, false);
  sfg_tensor* a_csr = nullptr;
  try {
    a_csr = coo_to_csc(ctx, at);
  } catch (...) {
    free_tensor(at);
    throw;
  }
  free_tensor(at);
  sfg_tensor* out = nullptr;
  try {
    out = row_compressed_to_coo(ctx, a_csr->ptr, nullptr, s->m, a_csr->idx, static_cast<const float*>(a_csr->val),
                                a_csr->nnz, s->m, s->n, false);
  } catch (...) {
    free_tensor(a_csr);
    throw;
  }
  free_tensor(a_csr);
  return out;
}


// The nonzero entries of an ELL or BELL tensor as a canonical COO (for
// operations whose result does not depend on zero slots, e.g. SpGEMM).
sfg_tensor* ell_nonzeros_to_coo(sfg_context* ctx, const sfg_tensor* s) {
  const bool bell = s->kind == SFG_BELL;
  const int64_t cells = bell ? s->k * s->nbr * s->rb * s->cb : s->k * s->m;
  sfg_tensor* tmp = make_coo(ctx, s->m, s->n, cells);
  auto* count = static_cast<unsigned long long*>(scratch(ctx, 64));
  SFG_CUDA(cudaMemsetAsync(count, 0, 8, ctx->stream));
  if (cells && bell)
    SFG_LAUNCH(k_bell_nonzeros, stream_grid(ctx, cells, kBlock, 1, 8), kBlock, 0, ctx->stream, s->idx,
               static_cast<const float*>(s->val), s->nbr, s->k * s->nbr, (int32_t)s->br, (int32_t)s->rb,
               (int32_t)s->cb, tmp->row, tmp->idx, static_cast<float*>(tmp->val), count);
  else if (cells)
    SFG_LAUNCH(k_ell_nonzeros, stream_grid(ctx, cells, kBlock, 1, 8), kBlock, 0, ctx->stream, s->idx,
               static_cast<const float*>(s->val), s->m, s->k, tmp->row, tmp->idx, static_cast<float*>(tmp->val),
               count);
  unsigned long long nz = 0;
  read_back(ctx, count, 8, &nz);
  sfg_tensor* out = nullptr;
  try {
    out = sort_coo(ctx, s->m, s->n, (int64_t)nz, tmp->row, tmp->idx, static_cast<const float*>(tmp->val), false);
  } catch (...) {
    free_tensor(tmp);
    throw;
  }
  free_tensor(tmp);
  return out;
}

namespace {

sfg_tensor* deep_copy(sfg_context* ctx, const sfg_tensor* s) {
  tensor_nnr(s);  // the copy must not share a pending read-back slot
  sfg_tensor* t = new sfg_tensor(*s);
  t->tc_plan = nullptr;
  t->tc_base = nullptr;
  t->tc_desc = nullptr;
  t->part[0] = t->part[1] = nullptr;
  t->row = t->ptr = t->idx = t->slots = t->ptr1 = nullptr;
  t->val = nullptr;
  auto dup = [&](const void* p, size_t bytes) -> void* {
    if (!p) return nullptr;
    void* q = dalloc(ctx, bytes);
    SFG_CUDA(cudaMemcpyAsync(q, p, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
    return q;
  };
  const size_t esz = s->dtype == SFG_BF16 ? 2 : 4;
  switch (s->kind) {
    case SFG_COO:
      t->row = static_cast<int32_t*>(dup(s->row, s->nnz * 4));
      t->idx = static_cast<int32_t*>(dup(s->idx, s->nnz * 4));
      t->val = dup(s->val, s->nnz * esz);
      break;
    case SFG_CSR:
      t->ptr = static_cast<int32_t*>(dup(s->ptr, (s->m + 1) * 4));
      t->idx = static_cast<int32_t*>(dup(s->idx, s->nnz * 4));
      t->val = dup(s->val, s->nnz * esz);
      break;
    case SFG_CSC:
      t->ptr = static_cast<int32_t*>(dup(s->ptr, (s->n + 1) * 4));
      t->idx = static_cast<int32_t*>(dup(s->idx, s->nnz * 4));
      t->val = dup(s->val, s->nnz * esz);
      break;
    case SFG_DCSR:
    case SFG_DCSC:
      t->row = static_cast<int32_t*>(dup(s->row, s->nnr * 4));  // resolved above
      t->ptr = static_cast<int32_t*>(dup(s->ptr, (s->nnr + 1) * 4));
      t->idx = static_cast<int32_t*>(dup(s->idx, s->nnz * 4));
      t->val = dup(s->val, s->nnz * esz);
      break;
    case SFG_BCSR:
      t->ptr = static_cast<int32_t*>(dup(s->ptr, (s->nbr + 1) * 4));
      t->idx = static_cast<int32_t*>(dup(s->idx, s->nnz * 4));
      t->val = dup(s->val, s->nnz * s->rb * s->cb * esz);
      break;
    case SFG_DIA:
      t->slots = static_cast<int32_t*>(dup(s->slots, s->k * 4));
      t->val = dup(s->val, s->k * s->m * esz);
      break;
    case SFG_CSB:
      t->ptr = static_cast<int32_t*>(dup(s->ptr, (s->nbr * s->nbc + 1) * 4));
      t->row = static_cast<int32_t*>(dup(s->row, s->nnz * 4));
      t->idx = static_cast<int32_t*>(dup(s->idx, s->nnz * 4));
      t->val = dup(s->val, s->nnz * esz);
      break;
    default:
      delete t;
      raise(SFG_ERR_UNSUPPORTED_SOURCE, "identity copy of this format");
  }
  return t;
}

}  // namespace

sfg_tensor* convert_from_compressed(sfg_context* ctx, const sfg_tensor* s, const sfg_format& dst) {
  if (s->kind == SFG_ELL || s->kind == SFG_BELL || s->kind == SFG_CISR || s->kind == SFG_CISRP)
    raise(SFG_ERR_UNSUPPORTED_SOURCE, "conversion from a format with indirect levels");
  if (s->kind == SFG_HYB || s->kind == SFG_HBELL)
    raise(SFG_ERR_UNSUPPORTED_SOURCE, "conversion from the hybrid pair");
  // planner.hpp:98-99: sources with a value layout are rejected
  if (s->kind == SFG_DOK || s->kind == SFG_LIL || s->kind == SFG_C2SR)
    raise(SFG_ERR_UNSUPPORTED_SOURCE, "conversion from a format with a value layout");
  // The reference expands a DIA source through its skewed map, so the
  // column level comes back with the interval [-(m-1), n+m-2] (and a CSB
  // source with its tile-grid extents and extra dangling nodes); the device
  // tensors keep [0, n-1] columns, so these sources are not converted.
  if (s->kind == SFG_DIA || s->kind == SFG_DIAV || s->kind == SFG_BDIA || s->kind == SFG_CSB)
    raise(SFG_ERR_UNSUPPORTED_SOURCE,
          "conversion from DIA / DIA-variant / BDIA / CSB: the reference's skewed / tile-grid level bounds are not "
          "held on the device");
  // From a column-major source the reference reaches DIA-variant's map by
  // Skew(1,0,-1) Skew(0,1,1), which widens the column level to
  // [-(m-1), n+m-2] (a panel of ndiag x (n + 2(m-1)) cells); the device's
  // DIA-variant keeps [0, n-1].
  if (dst.kind == SFG_DIAV && (s->kind == SFG_CSC || s->kind == SFG_DCSC))
    raise(SFG_ERR_UNSUPPORTED_SOURCE,
          "CSC / DCSC -> DIA-variant: the reference's skewed plan widens the column level to [-(m-1), n+m-2], "
          "not held on the device");
  const bool same = s->kind == dst.kind &&
                    (s->kind != SFG_BCSR || (s->br == dst.block_r && s->bc == dst.block_c && s->dtype == dst.value_dtype)) &&
                    (s->kind != SFG_CSB || (s->br == dst.block_r && s->bc == dst.block_c));
  if (same) return deep_copy(ctx, s);
  sfg_tensor* coo = nullptr;
  switch (s->kind) {
    case SFG_CSR:  // Trim(0) unless the target keeps the CSR structure
      coo = row_compressed_to_coo(ctx, s->ptr, nullptr, s->m, s->idx, static_cast<const float*>(s->val), s->nnz,
                                  s->m, s->n, dst.kind != SFG_CSR);
      break;
    case SFG_DCSR:
      coo = row_compressed_to_coo(ctx, s->ptr, s->row, tensor_nnr(s), s->idx, static_cast<const float*>(s->val), s->nnz,
                                  s->m, s->n, false);
      break;
    case SFG_CSC:
      coo = csc_to_coo(ctx, s, dst.kind != SFG_CSC);
      break;
    case SFG_DCSC:
      coo = dcsc_to_coo(ctx, s);
      break;
    case SFG_BCSR:
      coo = bcsr_to_coo(ctx, s);
      break;
    default:
      raise(SFG_ERR_UNSUPPORTED_SOURCE, "unsupported source format");
  }
  coo->has_zeros = -1;
  sfg_tensor* out = nullptr;
  try {
    if (coo->m <= 0 || coo->n <= 0) raise(SFG_ERR_INVALID_OPERATION, "empty bounds at extent-only level");
    switch (dst.kind) {
      case SFG_COO: out = coo_to_coo(ctx, coo); break;
      case SFG_CSR: out = coo_to_csr(ctx, coo); break;
      case SFG_CSC: out = coo_to_csc(ctx, coo); break;
      case SFG_DCSR: out = coo_to_dcsr(ctx, coo); break;
      case SFG_ELL: out = coo_to_ell(ctx, coo); break;
      case SFG_BCSR: out = coo_to_bcsr(ctx, coo, dst.block_r, dst.block_c, dst.value_dtype); break;
      case SFG_HYB: out = coo_to_hyb(ctx, coo, dst.threshold); break;
      case SFG_HBELL: out = coo_to_hbell(ctx, coo, dst.block_r, dst.threshold); break;
      case SFG_BELL: out = coo_to_bell(ctx, coo, dst.block_r); break;
      case SFG_DOK: out = coo_to_dok(ctx, coo); break;
      case SFG_LIL: out = coo_to_lil(ctx, coo); break;
      case SFG_DIA: out = coo_to_dia(ctx, coo); break;
      case SFG_DIAV: out = coo_to_dia(ctx, coo, true); break;
      case SFG_DCSC: out = coo_to_dcsc(ctx, coo); break;
      case SFG_CISR:
      case SFG_CISRP: out = coo_to_cisr(ctx, coo, dst.block_r, dst.kind == SFG_CISRP); break;
      case SFG_CSB: out = coo_to_csb(ctx, coo, dst.block_r, dst.block_c); break;
      case SFG_BDIA: out = coo_to_bdia(ctx, coo, dst.block_r); break;
      case SFG_C2SR: out = coo_to_c2sr(ctx, coo, dst.block_r); break;
      default: raise(SFG_ERR_INVALID_OPERATION, "unknown target");
    }
  } catch (...) {
    free_tensor(coo);
    throw;
  }
  free_tensor(coo);
  return out;
}

}  // namespace sfg
