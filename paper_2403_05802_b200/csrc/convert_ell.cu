// convert_ell.cu — the query-driven conversions: decompose by row count,
// COO -> ELL, and the hybrid ELL+COO pair.
//
// Reference semantics (paths relative to proj/include/sparseforge/):
//  * Sum query "sum(value) groupBy (d0,d1)->(d0) with value ne 0 -> 1"
//    (formats.hpp:20-23, query_engine.hpp:112-125): per-row count of
//    nonzero values over the dense row domain.
//  * decompose (decompose.hpp:30-63): rows whose count >= min_sum are
//    `selected`, the rest `remainder`; order is preserved.
//  * ELL = plan Sum(0) Enumerate(0) Sort Fill(1,PadPath) Merge(0)
//    (planner.hpp:218-249). Enumerate (query_engine.hpp:166-201 with
//    formats.hpp:25-28) gives a row's nonzeros slots 0..nz-1 in column order
//    and its explicit zeros nz, nz+1, ...; K = max slot + 1. Fill(1) pads
//    every (slot, row) cell without an entry with column 0 (the level's
//    lower bound) and value 0 (operators.hpp:203-226). Materialized
//    slot-major: L0 idx[K] = 0..K-1, L2 idx[K*M], val[K*M].
//  * hybrid: decompose, remainder -> ELL, selection -> COO.
//
// Device plan (all from row-sorted canonical COO):
//  1. k_row_ptr   : row pointers from the sorted row array (like CSR) and
//                   the per-row count of explicit zeros (atomics on zeros
//                   only, so zero-free inputs pay nothing).
//  2. k_row_scan  : per-row selection flag, single-pass look-back scan of the
//                   selected entry counts, K = max remainder row length.
//  3. k_split     : entries of selected rows -> COO (and, for decompose, the
//                   remainder -> COO), position = e - offset[row].
//  4. k_ell_fill  : thread per row writes its K slot-major cells (coalesced),
//                   gathering the row's remainder entries, padding the rest.
#include <cuda_bf16.h>

#include "devutil.cuh"
#include "internal.cuh"

namespace sfg {

namespace {

constexpr int kBlock = 256;
constexpr uint32_t kSelBit = 0x80000000u;

// --------------------------------------------------------- 1. row pointers
// A warp handles 128*kRowVec consecutive entries per iteration. kVals: the
// source may hold explicit zeros, so values are read too; a zero-free
// source reads rows only.
constexpr int kRowVec = 4;

template <bool kVals>
__global__ void __launch_bounds__(kBlock) k_row_ptr(const int32_t* __restrict__ row,
                                                     const float* __restrict__ val, int64_t nnz,
                                                     int32_t m, int32_t* __restrict__ ptr,
                                                     int32_t* __restrict__ zcnt,
                                                     int* __restrict__ any_zero) {
  constexpr int kChunk = 128 * kRowVec;
  __shared__ __align__(16) int32_t s_rows[kBlock / 32][kChunk];
  const int lane = threadIdx.x & 31;
  const int64_t nchunk = (nnz + kChunk - 1) / kChunk;
  const int64_t warps = (int64_t)gridDim.x * (kBlock / 32);
  bool saw_zero = false;
  // software pipeline: the next chunk's rows are in flight while this
  // chunk's row pointers are searched and written
  int64_t ch = (int64_t)blockIdx.x * (kBlock / 32) + (threadIdx.x >> 5);
  RowChunk<kRowVec> next;
  if (ch < nchunk) load_row_chunk(row, nnz, ch * kChunk, next);
  for (; ch < nchunk; ch += warps) {
    const int64_t base = ch * kChunk;
    RowChunk<kRowVec> c = next;
    if (ch + warps < nchunk) load_row_chunk(row, nnz, (ch + warps) * kChunk, next);
    if (kVals) {
#pragma unroll
      for (int g = 0; g < kRowVec; ++g) {
        int64_t e0 = base + 128 * g + 4 * lane;
        float x[4];
        if (c.full) {
          float4 vv = ld_stream(reinterpret_cast<const float4*>(val + e0));
          x[0] = vv.x; x[1] = vv.y; x[2] = vv.z; x[3] = vv.w;
        } else {
#pragma unroll
          for (int i = 0; i < 4; ++i) x[i] = e0 + i < nnz ? val[e0 + i] : 1.f;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (x[i] == 0.f) {
            atomicAdd(zcnt + c.r[g][i], 1);
            saw_zero = true;
          }
      }
    }
    chunk_row_ptr(c, nnz, base, m, s_rows[threadIdx.x >> 5], ptr);
  }
  if (kVals && __any_sync(kFull, saw_zero) && lane == 0) atomicOr(any_zero, 1);
}

// ------------------------------------------------------------ 2. row scan
// off[r] = selected ? kSelBit | (entries of unselected rows before r)
//                   : (entries of selected rows before r)
// so an entry e of row r lands at e - (off[r] & ~kSelBit) in its part.
constexpr int kScanItems = 16;
constexpr int kScanTile = kBlock * kScanItems;

struct ScanOut {
  int32_t nnz_sel;
  int32_t k_max;  // max entries over unselected rows
};

__global__ void __launch_bounds__(kBlock) k_row_scan(const int32_t* __restrict__ ptr,
                                                      const int32_t* __restrict__ zcnt,
                                                      int has_zeros, int32_t m, int64_t min_sum,
                                                      uint32_t* __restrict__ off,
                                                      int32_t* __restrict__ totals,
                                                      unsigned long long* __restrict__ status,
                                                      uint32_t epoch, ScanOut* __restrict__ out) {
  __shared__ uint32_t smem[34];
  __shared__ uint32_t slot;
  // The tile's row pointers / zero counts / outputs go through shared memory
  // (skewed by one word per 16 so the per-thread runs are conflict-free), so
  // every global access is coalesced.
  __shared__ int32_t sp[kScanTile + kScanTile / 16 + 2];
  __shared__ int32_t sz[kScanTile + kScanTile / 16 + 1];
  auto sk = [](int i) { return i + (i >> 4); };
  const int64_t tile0 = (int64_t)blockIdx.x * kScanTile;
  {
    // all loads in flight before the first shared store
    int32_t pv[kScanItems], zv[kScanItems];
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      int64_t r = tile0 + threadIdx.x + k * kBlock;
      pv[k] = r <= m ? ld_stream(ptr + r) : 0;
      zv[k] = (has_zeros && r < m) ? ld_stream(zcnt + r) : 0;
    }
    int32_t pend = 0;
    if (threadIdx.x == 0 && tile0 + kScanTile <= m) pend = __ldg(ptr + tile0 + kScanTile);
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      int i = threadIdx.x + k * kBlock;
      sp[sk(i)] = pv[k];
      sz[sk(i)] = zv[k];
    }
    if (threadIdx.x == 0) sp[sk(kScanTile)] = pend;
  }
  __syncthreads();
  const int t0 = threadIdx.x * kScanItems;
  const int64_t r0 = tile0 + t0;
  uint32_t cnt[kScanItems];
  uint32_t selmask = 0, sum = 0;
  int32_t kmax = 0;
  int32_t p_lo = sp[sk(t0)];
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    int64_t r = r0 + i;
    cnt[i] = 0;
    if (r < m) {
      int32_t p_hi = sp[sk(t0 + i + 1)];
      int32_t c = p_hi - p_lo;
      int32_t nz = has_zeros ? c - sz[sk(t0 + i)] : c;
      if (totals) totals[r] = nz;
      bool sel = (int64_t)nz >= min_sum;
      if (sel) {
        selmask |= 1u << i;
        sum += c;
      } else if (c > kmax) {
        kmax = c;
      }
      cnt[i] = c;
      p_lo = p_hi;
    }
  }
  uint32_t total;
  uint32_t excl = block_exclusive_scan<uint32_t, kBlock>(sum, smem, &total);
  kmax = warp_max(kmax);
  if ((threadIdx.x & 31) == 0 && kmax > 0) atomicMax(&out->k_max, kmax);
  uint32_t tp = lookback_prefix(status, epoch, blockIdx.x, total, &slot);
  uint32_t sel_before = tp + excl;
  int32_t p = sp[sk(t0)];
  uint32_t* so = reinterpret_cast<uint32_t*>(sz);  // reuse: per-row offsets
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    bool sel = (selmask >> i) & 1u;
    so[sk(t0 + i)] = sel ? (kSelBit | (uint32_t)(p - sel_before)) : sel_before;
    if (sel) sel_before += cnt[i];
    p += cnt[i];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kScanTile; i += kBlock)
    if (tile0 + i < m) off[tile0 + i] = so[sk(i)];
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) out->nnz_sel = (int32_t)(tp + total);
}

// ---------------------------------------------------------------- 3. split
constexpr int kSplitRun = 8;

#ifndef SFG_SPLIT_MINB
#define SFG_SPLIT_MINB 1  // config 2 conversion: 1 (64 registers) 0.437 ms; 5 -> 0.486 (spills)
#endif
__global__ void __launch_bounds__(kBlock, SFG_SPLIT_MINB) k_split(
    const int32_t* __restrict__ row, const int32_t* __restrict__ col,
    const float* __restrict__ val, int64_t nnz, const uint32_t* __restrict__ off,
    int32_t* __restrict__ srow, int32_t* __restrict__ scol, float* __restrict__ sval,
    int32_t* __restrict__ rrow, int32_t* __restrict__ rcol, float* __restrict__ rval) {
  // A warp owns 32*kSplitRun consecutive entries, lane-strided: at step i
  // lane l handles entry base + 32 i + l, so loads are coalesced and, since
  // consecutive entries of one part land at consecutive positions, so are
  // the stores (blocked per-thread runs scattered 4-byte stores 32 B apart,
  // which cost L2 partial-sector read-modify-writes). All loads of the
  // warp's chunk are issued before the first store.
  constexpr int R = kSplitRun;
  const int lane = threadIdx.x & 31;
  const int64_t span = 32 * R;
  const int64_t nchunk = (nnz + span - 1) / span;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nchunk; w += warps) {
    const int64_t base = w * span + lane;
    int r[R], c[R];
    float x[R];
    uint32_t o[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      int64_t e = base + 32 * i;
      bool ok = e < nnz;
      r[i] = ok ? ld_stream(row + e) : -1;
      c[i] = ok ? ld_stream(col + e) : 0;
      x[i] = ok ? ld_stream(val + e) : 0.f;
    }
#pragma unroll
    for (int i = 0; i < R; ++i) o[i] = r[i] >= 0 ? __ldg(off + r[i]) : 0u;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      if (r[i] < 0) continue;
      int64_t pos = base + 32 * i - (int64_t)(o[i] & ~kSelBit);
      if (o[i] & kSelBit) {
        srow[pos] = r[i];
        scol[pos] = c[i];
        sval[pos] = x[i];
      } else if (rrow) {
        rrow[pos] = r[i];
        rcol[pos] = c[i];
        rval[pos] = x[i];
      }
    }
  }
}

// ------------------------------------------------------------ 4. ELL fill
// Thread per row r: cells s*m + r for s < K. Unselected rows place their
// entries in Enumerate order (nonzeros, then explicit zeros); everything
// else is padding (column 0, value 0).
__global__ void __launch_bounds__(kBlock) k_ell_fill(const int32_t* __restrict__ ptr,
                                                      const uint32_t* __restrict__ off,
                                                      const int32_t* __restrict__ zcnt,
                                                      int has_zeros,
                                                      const int32_t* __restrict__ col,
                                                      const float* __restrict__ val, int32_t m,
                                                      int32_t k, int32_t* __restrict__ eidx,
                                                      float* __restrict__ evl) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < m;
       r += (int64_t)gridDim.x * blockDim.x) {
    int32_t s0 = __ldg(ptr + r), s1 = __ldg(ptr + r + 1);
    bool sel = off ? (__ldg(off + r) & kSelBit) != 0 : false;
    int32_t c = sel ? 0 : s1 - s0;
    int32_t z = (has_zeros && !sel) ? __ldg(zcnt + r) : 0;
    if (z == 0) {
      for (int s = 0; s < k; ++s) {
        int64_t cell = (int64_t)s * m + r;
        if (s < c) {
          eidx[cell] = __ldg(col + s0 + s);
          evl[cell] = __ldg(val + s0 + s);
        } else {
          eidx[cell] = 0;
          evl[cell] = 0.f;
        }
      }
    } else {
      int s = 0;
      for (int32_t e = s0; e < s1; ++e) {
        float v = __ldg(val + e);
        if (v != 0.f) {
          eidx[(int64_t)s * m + r] = __ldg(col + e);
          evl[(int64_t)s * m + r] = v;
          ++s;
        }
      }
      for (int32_t e = s0; e < s1; ++e) {
        float v = __ldg(val + e);
        if (v == 0.f) {
          eidx[(int64_t)s * m + r] = __ldg(col + e);
          evl[(int64_t)s * m + r] = v;
          ++s;
        }
      }
      for (; s < k; ++s) {
        eidx[(int64_t)s * m + r] = 0;
        evl[(int64_t)s * m + r] = 0.f;
      }
    }
  }
}

__global__ void k_iota(int32_t* __restrict__ p, int32_t n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = i;
}

// Shared front half: row pointers, zero counts, selection scan.
struct RowInfo {
  int32_t* ptr = nullptr;
  int32_t* zcnt = nullptr;
  uint32_t* off = nullptr;
  int has_zeros = 0;
  int64_t nnz_sel = 0;
  int64_t k = 0;
};

// defer: the sizes (nnz_sel, k, has_zeros) are read back asynchronously;
// call row_info_finish before using them (work that needs only the device
// arrays — k_split — can be enqueued in between).
RowInfo row_info(sfg_context* ctx, const sfg_tensor* s, int64_t min_sum, int32_t* totals, bool defer = false) {
  RowInfo ri;
  const int64_t m = s->m;
  // Explicit zeros only matter when the source may hold them: a tensor known
  // to be zero-free (from_coo checked it, or a generator built it) skips the
  // value stream and the per-row zero counts entirely.
  const bool zeros_possible = s->has_zeros != 0;
  ri.ptr = dalloc_n<int32_t>(ctx, m + 1);
  ri.zcnt = zeros_possible ? dalloc_n<int32_t>(ctx, m) : nullptr;
  ri.off = dalloc_n<uint32_t>(ctx, m);
  int tiles = (int)ceil_div(m, kScanTile);
  auto* status = lookback_status(ctx, tiles);
  auto* tail = static_cast<int32_t*>(scratch(ctx, 64));  // [any_zero, nnz_sel, k_max]
  SFG_CUDA(cudaMemsetAsync(tail, 0, 16, ctx->stream));
  if (zeros_possible) SFG_CUDA(cudaMemsetAsync(ri.zcnt, 0, m * sizeof(int32_t), ctx->stream));
  if (s->nnz == 0) {
    SFG_CUDA(cudaMemsetAsync(ri.ptr, 0, (m + 1) * sizeof(int32_t), ctx->stream));
  } else {
    int grid = stream_grid(ctx, ceil_div(s->nnz, 128 * kRowVec), kBlock / 32, 1, 8);
    if (zeros_possible)
      SFG_LAUNCH(k_row_ptr<true>, grid, kBlock, 0, ctx->stream, s->row, static_cast<const float*>(s->val),
                 s->nnz, (int32_t)m, ri.ptr, ri.zcnt, tail);
    else
      SFG_LAUNCH(k_row_ptr<false>, grid, kBlock, 0, ctx->stream, s->row, nullptr, s->nnz, (int32_t)m,
                 ri.ptr, ri.zcnt, tail);
  }
  // zcnt is exact (zeroed, incremented only for zero values), so the scan
  // subtracts it whenever it exists; the flag only selects the ELL fill's
  // slow path.
  SFG_LAUNCH(k_row_scan, tiles, kBlock, 0, ctx->stream, ri.ptr, ri.zcnt, zeros_possible ? 1 : 0, (int32_t)m,
             min_sum, ri.off, totals, status, ctx->epoch++, reinterpret_cast<ScanOut*>(tail + 1));
  if (defer) {
    read_back_start(ctx, tail, 16);
    return ri;
  }
  int32_t h[4];
  read_back(ctx, tail, 16, h);
  ri.has_zeros = h[0];
  ri.nnz_sel = h[1];
  ri.k = h[2];
  return ri;
}

void row_info_finish(sfg_context* ctx, RowInfo& ri) {
  int32_t h[4];
  read_back_wait(ctx, 16, h);
  ri.has_zeros = h[0];
  ri.nnz_sel = h[1];
  ri.k = h[2];
}

void free_row_info(sfg_context* ctx, RowInfo& ri) {
  dfree(ctx, ri.ptr);
  dfree(ctx, ri.zcnt);
  dfree(ctx, ri.off);
}

sfg_tensor* coo_part(sfg_context* ctx, int64_t m, int64_t n, int64_t nnz) {
  sfg_tensor* t = new_tensor(ctx, SFG_COO, m, n);
  t->nnz = nnz;
  t->row = dalloc_n<int32_t>(ctx, nnz);
  t->idx = dalloc_n<int32_t>(ctx, nnz);
  t->val = dalloc_n<float>(ctx, nnz);
  return t;
}

// ELL over all m rows from the canonical COO; rows flagged selected in `off`
// (or none when off == nullptr) are padding only.
sfg_tensor* ell_from(sfg_context* ctx, const sfg_tensor* s, const RowInfo& ri, bool use_sel) {
  sfg_tensor* t = new_tensor(ctx, SFG_ELL, s->m, s->n);
  t->k = ri.k;
  t->nnz = ri.k * s->m;
  t->slots = dalloc_n<int32_t>(ctx, ri.k);
  t->idx = dalloc_n<int32_t>(ctx, t->nnz);
  t->val = dalloc_n<float>(ctx, t->nnz);
  if (ri.k > 0) {
    SFG_LAUNCH(k_iota, 1, 256, 0, ctx->stream, t->slots, (int32_t)ri.k);
    SFG_LAUNCH(k_ell_fill, (int)ceil_div(s->m, kBlock), kBlock, 0, ctx->stream, ri.ptr,
               use_sel ? ri.off : nullptr, ri.zcnt, ri.has_zeros, s->idx,
               static_cast<const float*>(s->val), (int32_t)s->m, (int32_t)ri.k, t->idx,
               static_cast<float*>(t->val));
  }
  return t;
}

}  // namespace

void decompose_rows(sfg_context* ctx, const sfg_tensor* s, int64_t min_sum, sfg_tensor** sel,
                    sfg_tensor** rem, int32_t* totals) {
  RowInfo ri = row_info(ctx, s, min_sum, totals);
  sfg_tensor* a = coo_part(ctx, s->m, s->n, ri.nnz_sel);
  sfg_tensor* b = coo_part(ctx, s->m, s->n, s->nnz - ri.nnz_sel);
  a->has_zeros = b->has_zeros = s->has_zeros == 0 ? 0 : -1;
  if (s->nnz)
    SFG_LAUNCH(k_split, stream_grid(ctx, ceil_div(s->nnz, kSplitRun), kBlock, 1, 8), kBlock, 0, ctx->stream,
               s->row, s->idx, static_cast<const float*>(s->val), s->nnz, ri.off, a->row, a->idx,
               static_cast<float*>(a->val), b->row, b->idx, static_cast<float*>(b->val));
  free_row_info(ctx, ri);
  *sel = a;
  *rem = b;
}

sfg_tensor* coo_to_ell(sfg_context* ctx, const sfg_tensor* s) {
  // no row selected: every row goes to ELL, K = max row length
  RowInfo ri = row_info(ctx, s, INT64_MAX, nullptr);
  sfg_tensor* t = ell_from(ctx, s, ri, false);
  free_row_info(ctx, ri);
  return t;
}

sfg_tensor* coo_to_hyb(sfg_context* ctx, const sfg_tensor* s, int64_t min_sum) {
  // The split needs only the device offsets, so it is enqueued before the
  // host waits for the sizes: the read-back round trip overlaps the split
  // instead of idling the GPU. The COO part is allocated for every entry
  // (an upper bound) and its size set once known.
  //
  // The over-allocation (12 B for every entry not selected, held until the
  // tensor is freed) is only taken while it is small next to the device's
  // memory (an eighth of it); otherwise the sizes are waited for and the
  // COO part is allocated exactly. (Not decided on cudaMemGetInfo: that
  // call can block the host for milliseconds, and a decision flipping with
  // the momentary free memory would change the allocation sizes per call.)
  const size_t upper = 12 * static_cast<size_t>(s->nnz);
  const bool defer = upper <= (size_t(256) << 20) || upper <= ctx->total_mem / 8;
  RowInfo ri = row_info(ctx, s, min_sum, nullptr, defer);
  sfg_tensor* h = new_tensor(ctx, SFG_HYB, s->m, s->n);
  h->threshold = min_sum;
  h->part[1] = coo_part(ctx, s->m, s->n, defer ? s->nnz : ri.nnz_sel);
  h->part[1]->has_zeros = s->has_zeros == 0 ? 0 : -1;
  if (s->nnz)
    SFG_LAUNCH(k_split, stream_grid(ctx, ceil_div(s->nnz, kSplitRun), kBlock, 1, 8), kBlock, 0, ctx->stream,
               s->row, s->idx, static_cast<const float*>(s->val), s->nnz, ri.off, h->part[1]->row,
               h->part[1]->idx, static_cast<float*>(h->part[1]->val), nullptr, nullptr, nullptr);
  if (defer) row_info_finish(ctx, ri);
  h->part[1]->nnz = ri.nnz_sel;
  h->part[0] = ell_from(ctx, s, ri, true);
  free_row_info(ctx, ri);
  return h;
}

}  // namespace sfg
