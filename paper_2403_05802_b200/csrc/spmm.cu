// spmm.cu — C[M x nd] = A B over every materialized format (CUDA cores).
//
// Reference: run_kernel(spmm_kernel(), {A, B}) (kernel.hpp:236-384, 42-51):
// every stored slot (padding included) restores (d0, d1), is bounds-guarded,
// and for each d2 accumulates value * B[d1][d2] into C[d0][d2]. Here a warp
// owns a row (or a row-sorted run of entries) and its lanes own 32*V
// consecutive output columns: each stored entry is broadcast across the
// warp and multiplies one coalesced row of B. fp32 accumulate; B may be
// fp32 or bf16. The BCSR tensor-core path lives in bcsr_tc.cu.
#include <cuda_bf16.h>

#include <algorithm>
#include <climits>
#include <cstdlib>

#include "async.cuh"
#include "devutil.cuh"
#include "internal.cuh"

namespace sfg {

namespace {

constexpr int kBlock = 256;

template <typename TB>
struct BRow;

template <>
struct BRow<float> {
  template <int V>
  __device__ __forceinline__ static void load(const float* __restrict__ p, float (&v)[V]) {
    if constexpr (V == 4) {
      float4 q = __ldg(reinterpret_cast<const float4*>(p));
      v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
    } else if constexpr (V == 2) {
      float2 q = __ldg(reinterpret_cast<const float2*>(p));
      v[0] = q.x; v[1] = q.y;
    } else {
#pragma unroll
      for (int i = 0; i < V; ++i) v[i] = __ldg(p + i);
    }
  }
};

template <>
struct BRow<__nv_bfloat16> {
  template <int V>
  __device__ __forceinline__ static void load(const __nv_bfloat16* __restrict__ p, float (&v)[V]) {
    if constexpr (V == 4) {
      uint2 q = __ldg(reinterpret_cast<const uint2*>(p));
      v[0] = __uint_as_float(q.x << 16); v[1] = __uint_as_float(q.x & 0xffff0000u);
      v[2] = __uint_as_float(q.y << 16); v[3] = __uint_as_float(q.y & 0xffff0000u);
    } else if constexpr (V == 2) {
      uint32_t q = __ldg(reinterpret_cast<const unsigned int*>(p));
      v[0] = __uint_as_float(q << 16); v[1] = __uint_as_float(q & 0xffff0000u);
    } else {
#pragma unroll
      for (int i = 0; i < V; ++i) v[i] = __bfloat162float(p[i]);
    }
  }
};

// Geometry of the dense operands shared by every kernel.
struct Dense {
  const void* b;
  int64_t ldb;
  float* c;
  int64_t ldc;
  int32_t nd;
  int acc;        // non-atomic row stores add to C (accumulate, or C was zeroed first)
  int keep = 0;   // the caller's accumulate flag (C holds input to add to)
  int64_t zero_m = 0;  // DCSR, not accumulating: rows of C (the gaps are zeroed in the kernel)
};

// DCSR without accumulate: the rows of C between stored row p - 1 and
// stored row p (and, for the last stored row, up to M) hold no entry; the
// warp that owns row p zeroes its column chunk of them.
template <int V>
__device__ __forceinline__ void zero_gap_before(const Dense& d, const int32_t* __restrict__ rows, int64_t p,
                                                int64_t nrows, int c0) {
  if (!d.zero_m || !rows) return;
  const int64_t lo = p == 0 ? 0 : (int64_t)__ldg(rows + p - 1) + 1;
  const int64_t hi = p < nrows ? (int64_t)__ldg(rows + p) : d.zero_m;
  for (int64_t r = lo; r < hi; ++r)
#pragma unroll
    for (int i = 0; i < V; ++i)
      if (c0 + i < d.nd) d.c[r * d.ldc + c0 + i] = 0.f;
}

// B[col][cols of this lane] for the lane's column chunk.
template <typename TB, int V>
__device__ __forceinline__ void load_brow(const Dense& d, int col, int c0, bool vec, float (&v)[V]) {
  const TB* brow = static_cast<const TB*>(d.b) + (int64_t)col * d.ldb + c0;
  if (vec) {
    BRow<TB>::template load<V>(brow, v);
  } else {
#pragma unroll
    for (int i = 0; i < V; ++i) v[i] = c0 + i < d.nd ? (float)brow[i] : 0.f;
  }
}

template <int V>
__device__ __forceinline__ void store_vec(float* p, const float (&v)[V]) {
  if constexpr (V == 4) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  } else if constexpr (V == 2) {
    *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
  } else {
#pragma unroll
    for (int i = 0; i < V; ++i) p[i] = v[i];
  }
}

// Accumulate `val * B[col][cols of this lane]` for the lane's column chunk.
template <typename TB, int V>
__device__ __forceinline__ void fma_row(const Dense& d, int col, float val, int c0, bool vec,
                                        float (&acc)[V]) {
  const TB* brow = static_cast<const TB*>(d.b) + (int64_t)col * d.ldb + c0;
  float v[V];
  if (vec) {
    BRow<TB>::template load<V>(brow, v);
  } else {
#pragma unroll
    for (int i = 0; i < V; ++i) v[i] = c0 + i < d.nd ? (float)brow[i] : 0.f;
  }
#pragma unroll
  for (int i = 0; i < V; ++i) acc[i] = fmaf(val, v[i], acc[i]);
}

template <int V>
__device__ __forceinline__ void store_row(const Dense& d, int64_t row, int c0, bool atomic,
                                          const float (&acc)[V]) {
  float* crow = d.c + row * d.ldc + c0;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    if (c0 + i >= d.nd) break;
    if (atomic) atomicAdd(crow + i, acc[i]);
    else crow[i] = d.acc ? crow[i] + acc[i] : acc[i];
  }
}

// -------------------------------------------------------------- CSR/DCSR
// rows == nullptr: CSR (row p is row p); otherwise DCSR (row = rows[p]).
template <typename TB, int V>
__global__ void __launch_bounds__(kBlock) k_spmm_rows(const int32_t* __restrict__ rows,
                                                       const int32_t* __restrict__ ptr,
                                                       const int32_t* __restrict__ col,
                                                       const float* __restrict__ val, int64_t nrows,
                                                       Dense d) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int chunks = (d.nd + 32 * V - 1) / (32 * V);
  const bool vec_ok = (d.nd % (32 * V) == 0) && (d.ldb % V == 0);
  for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nrows * chunks;
       w += warps) {
    int64_t p = w / chunks;
    int c0 = (int)(w - p * chunks) * 32 * V + lane * V;
    int s = __ldg(ptr + p), e = __ldg(ptr + p + 1);
    float acc[V];
#pragma unroll
    for (int i = 0; i < V; ++i) acc[i] = 0.f;
    for (int base = s; base < e; base += 32) {
      int k = base + lane;
      int mc = k < e ? ld_stream(col + k) : 0;
      float mv = k < e ? ld_stream(val + k) : 0.f;
      int cnt = min(32, e - base);
      int j = 0;
      for (; j + 2 <= cnt; j += 2) {
        int c1 = __shfl_sync(kFull, mc, j), c2 = __shfl_sync(kFull, mc, j + 1);
        float v1 = __shfl_sync(kFull, mv, j), v2 = __shfl_sync(kFull, mv, j + 1);
        fma_row<TB, V>(d, c1, v1, c0, vec_ok, acc);
        fma_row<TB, V>(d, c2, v2, c0, vec_ok, acc);
      }
      if (j < cnt) fma_row<TB, V>(d, __shfl_sync(kFull, mc, j), __shfl_sync(kFull, mv, j), c0, vec_ok, acc);
    }
    int64_t r = rows ? __ldg(rows + p) : p;
    store_row<V>(d, r, c0, false, acc);
    zero_gap_before<V>(d, rows, p, nrows, c0);
    if (p == nrows - 1) zero_gap_before<V>(d, rows, nrows, nrows, c0);
  }
}

// Merge-path CSR (load balanced by rows + entries, so one row of a million
// entries does not serialise the kernel). The (row ends, entries) merge
// sequence of length m + nnz is cut into chunks of kMergeItems; a first
// kernel finds every cut's (row, entry) coordinate by binary search
// (Merrill & Garland's merge-path), then a warp per chunk walks its entries
// in order. Every row of C is written exactly once, by the chunk holding the
// row's end item: rows with no entry are zeroed there (no memset of C), a
// completed row stores this chunk's part of it. A row still open at the end
// of a chunk leaves its partial sum in a carry slot (one per chunk), and
// carry_fix adds the carries of each row in chunk order afterwards —
// no atomics, so C is bit-identical from run to run (the reference reduces
// its thread partials in worker order for the same reason, kernel.hpp:370-384).
constexpr int kMergeItems = 1024;

__global__ void k_merge_cuts(const int32_t* __restrict__ ptr, int64_t m, int64_t nnz, int64_t ncuts,
                             int2* __restrict__ cuts) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < ncuts; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t dgl = std::min<int64_t>(q * kMergeItems, m + nnz);
    int64_t lo = dgl > nnz ? dgl - nnz : 0, hi = dgl < m ? dgl : m;
    while (lo < hi) {  // rows consumed before the diagonal: row ends ptr[i+1] <= entries consumed
      const int64_t mid = (lo + hi) >> 1;
      if ((int64_t)__ldg(ptr + mid + 1) <= dgl - mid - 1) lo = mid + 1;
      else hi = mid;
    }
    cuts[q] = make_int2((int)lo, (int)(dgl - lo));
  }
}

// Carry slots of the merge-path walkers: row[q] = the row open at the end of
// chunk q (-1: none), val[q * nd + c] its partial sum over the chunk.
struct Carry {
  int32_t* row;
  float* val;
};

// A warp walks one merge-path chunk for one chunk of output columns. The
// warp splits into G lane groups of L = 32 / G lanes; a group covers L·V
// output columns (V per lane) and takes one entry per load instruction, so
// a narrow dense operand (nd = 32: G = 4 groups of 8 lanes × float4) still
// has G entries per warp instruction. Each group keeps a partial sum of the
// current row; closing a row reduces the G partials with lane shuffles and
// group 0 stores. While a step's kStep = G·kU entries all lie inside the
// current row the step is branch-free, its B rows loaded back to back.
// kVec: nd a multiple of L·V, vector-aligned B and C (no column guards).
#ifndef SFG_MERGE_MINB
#define SFG_MERGE_MINB 5  // CTAs per SM the register budget is sized for (config 5 SpMM: 5 -> 24.1 ms, 4 -> 25.1, 3 -> 25.1)
#endif
// S: entry stride (1 separate idx / val arrays; 2 LIL records {col, val}).
template <typename TB, int G, int V, int kU, bool kVec, bool kOne, int kMinB, int S>
__global__ void __launch_bounds__(kBlock, kMinB) k_spmm_merge(const int32_t* __restrict__ ptr,
                                                               const int32_t* __restrict__ col,
                                                               const float* __restrict__ val,
                                                               const int2* __restrict__ cuts, int64_t nchunks,
                                                               int32_t m, Dense d, Carry cy) {
  constexpr int L = 32 / G;  // lanes per group
  constexpr int kStep = G * kU;
  static_assert(G * L == 32 && kStep <= 32, "groups tile the warp");
  static_assert(kVec || V == 1, "guarded columns are scalar");
  const int lane = threadIdx.x & 31, grp = lane / L, sub = lane % L;
  const int ccols = kOne ? 1 : (d.nd + L * V - 1) / (L * V);  // column chunks (kOne: nd == L V)
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nchunks * ccols; w += warps) {
    const int64_t q = kOne ? w : w / ccols;
    const int cc = kOne ? 0 : (int)(w - q * ccols);
    const int c0 = cc * L * V + sub * V;
    const bool live_col = kVec || c0 < d.nd;
    const int2 a = __ldg(cuts + q), b = __ldg(cuts + q + 1);
    int i = a.x;
    const int j0 = a.y, j1 = b.y;
    // row-end window: lane t holds ptr[wb + t + 1] (rows past m: INT_MAX)
    int wb = i;
    int pw = wb + lane < m ? __ldg(ptr + wb + lane + 1) : INT_MAX;
    int row_end = __shfl_sync(kFull, pw, 0);
    float acc[V];
#pragma unroll
    for (int k = 0; k < V; ++k) acc[k] = 0.f;
    bool any = false;  // entries of row i seen in this chunk
    auto reduce = [&]() {
#pragma unroll
      for (int o = L; o < 32; o <<= 1)
#pragma unroll
        for (int k = 0; k < V; ++k) acc[k] += __shfl_xor_sync(kFull, acc[k], o);
    };
    auto put = [&](int64_t r, float (&x)[V]) {  // C[r][this lane's columns] = x (+ C with accumulate)
      float* crow = d.c + r * d.ldc + c0;
      if constexpr (kVec) {
        if (d.keep) {
          float o[V];
          BRow<float>::template load<V>(crow, o);
#pragma unroll
          for (int k = 0; k < V; ++k) x[k] += o[k];
        }
        store_vec<V>(crow, x);
      } else {
        if (live_col) crow[0] = d.keep ? crow[0] + x[0] : x[0];
      }
    };
    // Row i is complete (its end item lies in this chunk at or before entry
    // position `at`): store it and move to the first row ending after `at`
    // (rows from b.x on are closed by later chunks). The empty rows passed
    // over are zeroed once the chunk is done.
    const int lim = b.x;
    auto close = [&](int at) {
      reduce();
      if (grp == 0 && (any || !d.keep)) put(i, acc);
#pragma unroll
      for (int k = 0; k < V; ++k) acc[k] = 0.f;
      any = false;
      int r = i + 1;
      for (;;) {
        if (r - wb >= 32) {
          wb = r;
          pw = wb + lane < m ? __ldg(ptr + wb + lane + 1) : INT_MAX;
        }
        const unsigned past = __ballot_sync(kFull, pw > at) & (~0u << (r - wb));
        r = past ? wb + __ffs(past) - 1 : wb + 32;
        if (past || r >= lim) break;
      }
      i = min(r, lim);
      if (i - wb >= 32) {
        wb = i;
        pw = wb + lane < m ? __ldg(ptr + wb + lane + 1) : INT_MAX;
      }
      row_end = __shfl_sync(kFull, pw, i - wb);
    };
    for (int base = j0; base < j1; base += 32) {
      const int e = base + lane;
      int mc = 0;  // past the chunk: col 0, value 0
      float mv = 0.f;
      if (e < j1) ld_entry<S>(col, val, e, mc, mv);
      const int cnt = min(32, j1 - base);
      for (int t0 = 0; t0 < cnt; t0 += kStep) {
        const int last = base + min(t0 + kStep, cnt) - 1;
        // the step's B rows, entry t0 + u G + grp in group grp (past cnt:
        // B row 0, selected away), all loads in flight at once
        float v[kU][V];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int ck = __shfl_sync(kFull, mc, (t0 + u * G + grp) & 31);
          const TB* brow = static_cast<const TB*>(d.b) + (int64_t)ck * d.ldb + c0;
          if constexpr (kVec) {
            BRow<TB>::template load<V>(brow, v[u]);
          } else {
            v[u][0] = live_col ? (float)brow[0] : 0.f;
          }
        }
        if (last < row_end) {
          // fast path: the whole step is in row i
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            const bool live = t0 + u * G + grp < cnt;
            const float ak = __shfl_sync(kFull, mv, (t0 + u * G + grp) & 31);
#pragma unroll
            for (int k = 0; k < V; ++k) acc[k] = fmaf(ak, live ? v[u][k] : 0.f, acc[k]);
          }
          any = true;
        } else {
          // a row ends inside the step: entry by entry in order, closing
          // rows as they end; the owning group adds its preloaded row
          {
#pragma unroll
            for (int u = 0; u < kU; ++u)
#pragma unroll
              for (int gg = 0; gg < G; ++gg) {
                const int t = t0 + u * G + gg;
                if (t < cnt) {
                  const int j = base + t;
                  if (j >= row_end) close(j);
                  const float ak = __shfl_sync(kFull, mv, t);
                  if (grp == gg) {
#pragma unroll
                    for (int k = 0; k < V; ++k) acc[k] = fmaf(ak, v[u][k], acc[k]);
                  }
                  any = true;
                }
              }
          }
        }
      }
    }
    // rows ending at the chunk's end: complete here
    if (i < b.x) close(j1);
    // rows of this chunk without entries (ptr[r] == ptr[r + 1]) are zero
    if (!d.keep) {
      float z[V];
#pragma unroll
      for (int k = 0; k < V; ++k) z[k] = 0.f;
      for (int r0 = a.x; r0 < b.x; r0 += 32) {
        const int r = r0 + lane;
        const int hi = r < b.x ? __ldg(ptr + r + 1) : 0;
        const int lo = r < b.x ? __ldg(ptr + r) : 1;
        unsigned empty = __ballot_sync(kFull, hi == lo);
        while (empty) {  // G empty rows at a time, one per group
          int pick = -1;
#pragma unroll
          for (int g2 = 0; g2 < G; ++g2) {
            if (empty) {
              const int f = __ffs(empty) - 1;
              if (g2 == grp) pick = f;
              empty &= empty - 1;
            }
          }
          if (pick >= 0) put(r0 + pick, z);
        }
      }
    }
    // the row left open: its partial goes to the carry slot
    if (any) {
      reduce();
      if (grp == 0 && live_col) {
        float* cv = cy.val + q * d.nd + c0;
        if constexpr (kVec) {
          store_vec<V>(cv, acc);
        } else {
          cv[0] = acc[0];
        }
      }
    }
    if (cc == 0 && lane == 0) cy.row[q] = any ? i : -1;
  }
}


// Short rows (DCSR / CSR, <= 8 entries per row on average): a warp owns R
// consecutive stored rows, whose entries are one contiguous range. Lanes
// fetch 32 entries (col, val, local row) at a time, then the warp issues
// the B-row loads of kK entries back to back before consuming them in
// order — kK independent 32·V-wide gathers in flight per warp rather than
// one per row — flushing each row as the local row index moves past it.
// kVec: nd a multiple of 32 V and both leading dimensions multiples of V
// (vector loads / stores, no column guards) — chosen at launch.
template <typename TB, int V, int R, int kK, bool kVec>
__global__ void __launch_bounds__(kBlock) k_spmm_rows_batch(const int32_t* __restrict__ rows,
                                                             const int32_t* __restrict__ ptr,
                                                             const int32_t* __restrict__ col,
                                                             const float* __restrict__ val,
                                                             int64_t nrows, Dense d) {
  static_assert(R < 32 && kK <= 32, "row group and batch fit a warp");
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int chunks = (d.nd + 32 * V - 1) / (32 * V);
  constexpr bool vec_ok = kVec, vec_c = kVec;
  const bool gaps = d.zero_m && rows;  // DCSR, not accumulating: zero the rows between stored rows
  const int64_t groups = (nrows + R - 1) / R;
  for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < groups * chunks; w += warps) {
    const int64_t g = w / chunks;
    const int c0 = (int)(w - g * chunks) * 32 * V + lane * V;
    const int64_t p0 = g * R;
    const int nr = nrows - p0 < R ? (int)(nrows - p0) : R;
    const int pv = lane <= nr ? __ldg(ptr + p0 + lane) : 0;
    const int beg = __shfl_sync(kFull, pv, 0), end = __shfl_sync(kFull, pv, nr);
    // lane i < nr: output row of stored row p0 + i (and the one before it)
    const int orow = lane < nr ? (rows ? __ldg(rows + p0 + lane) : (int)(p0 + lane)) : 0;
    float acc[V];
#pragma unroll
    for (int i = 0; i < V; ++i) acc[i] = 0.f;
    int cur = 0;  // local row being accumulated
    auto store_cur = [&]() {
      float* crow = d.c + (int64_t)__shfl_sync(kFull, orow, cur) * d.ldc + c0;
      if (vec_c) {
        if (d.acc) {
          float o[V];
          BRow<float>::template load<V>(crow, o);
#pragma unroll
          for (int i = 0; i < V; ++i) acc[i] += o[i];
        }
        store_vec<V>(crow, acc);
      } else {
#pragma unroll
        for (int i = 0; i < V; ++i)
          if (c0 + i < d.nd) crow[i] = d.acc ? crow[i] + acc[i] : acc[i];
      }
#pragma unroll
      for (int i = 0; i < V; ++i) acc[i] = 0.f;
    };
    for (int base = beg; base < end; base += 32) {
      const int e = base + lane;
      const int mc = e < end ? ld_stream(col + e) : 0;
      const float mv = e < end ? ld_stream(val + e) : 0.f;
      int mr = 0;
#pragma unroll
      for (int i = 1; i < R; ++i) {
        const int b = __shfl_sync(kFull, pv, i);
        mr += (i < nr && b <= e) ? 1 : 0;
      }
      const int cnt = min(32, end - base);
      for (int k0 = 0; k0 < cnt; k0 += kK) {
        float v[kK][V];
        // past the batch end the lanes hold col 0 (a valid B row): the
        // loads are unconditional and the dead values are selected away, so
        // the batch has no per-entry branches besides the row flush
#pragma unroll
        for (int k = 0; k < kK; ++k) load_brow<TB, V>(d, __shfl_sync(kFull, mc, (k0 + k) & 31), c0, vec_ok, v[k]);
#pragma unroll
        for (int k = 0; k < kK; ++k) {
          const bool live = k0 + k < cnt;
          const int rk = __shfl_sync(kFull, mr, (k0 + k) & 31);
          const float ak = __shfl_sync(kFull, mv, (k0 + k) & 31);
          for (; cur < rk; ++cur) store_cur();  // rk of a dead slot is the last live row
#pragma unroll
          for (int i = 0; i < V; ++i) acc[i] = fmaf(ak, live ? v[k][i] : 0.f, acc[i]);
        }
      }
    }
    for (; cur < nr; ++cur) store_cur();
    if (gaps) {
      // rows with no entry before each stored row of the group (and after
      // the last stored row of the matrix) are zeroed here
      const int prev = lane == 0 ? (p0 == 0 ? -1 : __ldg(rows + p0 - 1)) : 0;
      int lo = __shfl_up_sync(kFull, orow, 1);
      if (lane == 0) lo = prev;
      const bool last = p0 + nr == nrows;
      for (int i = 0; i <= nr; ++i) {
        // gap before stored row i: (row of i - 1, row of i); i == nr: the
        // tail after the matrix's last stored row, up to M
        const int64_t a0 = (int64_t)__shfl_sync(kFull, lo, i) + 1;
        const int64_t a1 = i < nr ? (int64_t)__shfl_sync(kFull, orow, i) : (last ? d.zero_m : a0);
        for (int64_t r = a0; r < a1; ++r) {
          float* crow = d.c + r * d.ldc + c0;
          if (vec_c) {
            float z[V];
#pragma unroll
            for (int q = 0; q < V; ++q) z[q] = 0.f;
            store_vec<V>(crow, z);
          } else {
#pragma unroll
            for (int q = 0; q < V; ++q)
              if (c0 + q < d.nd) crow[q] = 0.f;
          }
        }
      }
    }
  }
}

// ------------------------------------------------------------------- ELL
template <typename TB, int V>
__global__ void __launch_bounds__(kBlock) k_spmm_ell(const int32_t* __restrict__ idx,
                                                      const float* __restrict__ val, int32_t m,
                                                      int32_t k, Dense d) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int chunks = (d.nd + 32 * V - 1) / (32 * V);
  const bool vec_ok = (d.nd % (32 * V) == 0) && (d.ldb % V == 0);
  for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < (int64_t)m * chunks;
       w += warps) {
    int64_t r = w / chunks;
    int c0 = (int)(w - r * chunks) * 32 * V + lane * V;
    float acc[V];
#pragma unroll
    for (int i = 0; i < V; ++i) acc[i] = 0.f;
    for (int s = 0; s < k; ++s) {
      int64_t cell = (int64_t)s * m + r;
      fma_row<TB, V>(d, __ldg(idx + cell), __ldg(val + cell), c0, vec_ok, acc);
    }
    store_row<V>(d, r, c0, false, acc);
  }
}

// ------------------------------------------------------------------- DIA
template <typename TB, int V>
__global__ void __launch_bounds__(kBlock) k_spmm_dia(const int32_t* __restrict__ diags,
                                                      const float* __restrict__ val, int64_t m, int64_t n,
                                                      int64_t k, bool by_col, Dense d) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int chunks = (d.nd + 32 * V - 1) / (32 * V);
  const bool vec_ok = (d.nd % (32 * V) == 0) && (d.ldb % V == 0);
  for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < m * chunks; w += warps) {
    const int64_t r = w / chunks;
    const int c0 = (int)(w - r * chunks) * 32 * V + lane * V;
    float acc[V];
#pragma unroll
    for (int i = 0; i < V; ++i) acc[i] = 0.f;
    for (int64_t q = 0; q < k; ++q) {
      const int64_t c = r + __ldg(diags + q);
      if (c >= 0 && c < n) fma_row<TB, V>(d, (int)c, __ldg(val + (by_col ? q * n + c : q * m + r)), c0, vec_ok, acc);
    }
    store_row<V>(d, r, c0, false, acc);
  }
}

// ------------------------------------------------------------------ BDIA
template <typename TB, int V>
__global__ void __launch_bounds__(kBlock) k_spmm_bdia(const int32_t* __restrict__ ptr,
                                                       const int32_t* __restrict__ diags,
                                                       const float* __restrict__ val, int64_t m, int64_t n,
                                                       int32_t b, int32_t rb, Dense d) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int chunks = (d.nd + 32 * V - 1) / (32 * V);
  const bool vec_ok = (d.nd % (32 * V) == 0) && (d.ldb % V == 0);
  for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < m * chunks; w += warps) {
    const int64_t r = w / chunks, br = r / b, ri = r - br * b;
    const int c0 = (int)(w - r * chunks) * 32 * V + lane * V;
    float acc[V];
#pragma unroll
    for (int i = 0; i < V; ++i) acc[i] = 0.f;
    for (int32_t q = __ldg(ptr + br); q < __ldg(ptr + br + 1); ++q) {
      const int64_t c = r + __ldg(diags + q);
      if (c >= 0 && c < n) fma_row<TB, V>(d, (int)c, __ldg(val + (int64_t)q * rb + ri), c0, vec_ok, acc);
    }
    store_row<V>(d, r, c0, false, acc);
  }
}

// ------------------------------------------------------------------- COO
// A warp owns 32*kCooIters consecutive row-sorted entries; it accumulates a
// row while the row stays the same and stores it when the row changes. A row
// belongs to the chunk holding its last entry (C was zeroed first, or holds
// the accumulate input, so that chunk adds its part with a plain store); a
// row continuing into the next chunk leaves its partial in the chunk's carry
// slot, added in chunk order by carry_fix — no atomics.
constexpr int kCooIters = 4;

// S: entry stride (1 separate arrays; 3 DOK records {row, col, val}).
template <typename TB, int V, int S>
__global__ void __launch_bounds__(kBlock) k_spmm_coo(const int32_t* __restrict__ row,
                                                      const int32_t* __restrict__ col,
                                                      const float* __restrict__ val, int64_t nnz,
                                                      Dense d, Carry cy) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int chunks = (d.nd + 32 * V - 1) / (32 * V);
  const bool vec_ok = (d.nd % (32 * V) == 0) && (d.ldb % V == 0);
  const int64_t span = 32 * kCooIters;
  const int64_t nchunks = (nnz + span - 1) / span;
  for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nchunks * chunks;
       w += warps) {
    int64_t q = w / chunks;
    const int cc = (int)(w - q * chunks);
    int c0 = cc * 32 * V + lane * V;
    int64_t e0 = q * span, e1 = min(nnz, e0 + span);
    int cur = __ldg(row + e0 * S);
    float acc[V];
#pragma unroll
    for (int i = 0; i < V; ++i) acc[i] = 0.f;
    for (int64_t base = e0; base < e1; base += 32) {
      int64_t k = base + lane;
      int mr = k < e1 ? __ldg(row + k * S) : -1;
      int mc = k < e1 ? __ldg(col + k * S) : 0;
      float mv = k < e1 ? __ldg(val + k * S) : 0.f;
      int cnt = (int)(e1 - base < 32 ? e1 - base : 32);
      for (int j = 0; j < cnt; ++j) {
        int rj = __shfl_sync(kFull, mr, j);
        if (rj != cur) {
          store_row<V>(d, cur, c0, false, acc);
#pragma unroll
          for (int i = 0; i < V; ++i) acc[i] = 0.f;
          cur = rj;
        }
        fma_row<TB, V>(d, __shfl_sync(kFull, mc, j), __shfl_sync(kFull, mv, j), c0, vec_ok, acc);
      }
    }
    const int next = e1 < nnz ? __ldg(row + e1 * S) : -1;
    if (cur != next) {
      store_row<V>(d, cur, c0, false, acc);
    } else {
#pragma unroll
      for (int i = 0; i < V; ++i)
        if (c0 + i < d.nd) cy.val[q * d.nd + c0 + i] = acc[i];
    }
    if (cc == 0 && lane == 0) cy.row[q] = cur != next ? -1 : cur;
  }
}

// ------------------------------------------------------------------- CSC
template <typename TB, int V>
__global__ void __launch_bounds__(kBlock) k_spmm_csc(const int32_t* __restrict__ ptr,
                                                      const int32_t* __restrict__ rowi,
                                                      const float* __restrict__ val, int32_t n,
                                                      Dense d) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int chunks = (d.nd + 32 * V - 1) / (32 * V);
  const bool vec_ok = (d.nd % (32 * V) == 0) && (d.ldb % V == 0);
  for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < (int64_t)n * chunks;
       w += warps) {
    int64_t c = w / chunks;
    int c0 = (int)(w - c * chunks) * 32 * V + lane * V;
    int s = __ldg(ptr + c), e = __ldg(ptr + c + 1);
    if (s == e) continue;
    float b[V], zero[V];
#pragma unroll
    for (int i = 0; i < V; ++i) zero[i] = 0.f, b[i] = 0.f;
    fma_row<TB, V>(d, (int)c, 1.f, c0, vec_ok, b);
    for (int k = s; k < e; ++k) {
      float v = __ldg(val + k);
      float a[V];
#pragma unroll
      for (int i = 0; i < V; ++i) a[i] = v * b[i];
      store_row<V>(d, __ldg(rowi + k), c0, true, a);
    }
    (void)zero;
  }
}

// ------------------------------------------------------------------ BCSR
// Warp per (block row, column chunk): lanes keep rb accumulators (one per
// row of the block row) for their V columns; every stored slot of every
// block is applied; rows/cols past M/N are guarded out (kernel.hpp:290-302).
// kBell: BELL cells — block row b holds the K slots k * nbr + b (padding:
// block column 0, a zero block), no ptr.
template <typename TB, typename TA, int V, int RB, bool kBell>
__global__ void __launch_bounds__(kBlock) k_spmm_bcsr(const int32_t* __restrict__ ptr,
                                                       const int32_t* __restrict__ bcol,
                                                       const TA* __restrict__ val, int64_t nbr,
                                                       int32_t m, int32_t n, int32_t br, int32_t bc,
                                                       int32_t rb, int32_t cb, Dense d, int64_t kslots) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int chunks = (d.nd + 32 * V - 1) / (32 * V);
  const bool vec_ok = (d.nd % (32 * V) == 0) && (d.ldb % V == 0);
  for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nbr * chunks;
       w += warps) {
    int64_t b = w / chunks;
    int c0 = (int)(w - b * chunks) * 32 * V + lane * V;
    float acc[RB][V];
#pragma unroll
    for (int i = 0; i < RB; ++i)
#pragma unroll
      for (int v = 0; v < V; ++v) acc[i][v] = 0.f;
    const int64_t s = kBell ? 0 : __ldg(ptr + b), e = kBell ? kslots : __ldg(ptr + b + 1);
    for (int64_t kk = s; kk < e; ++kk) {
      const int64_t k = kBell ? kk * nbr + b : kk;
      int colbase = __ldg(bcol + k) * bc;
      const TA* blk = val + k * rb * cb;
      for (int j = 0; j < cb; ++j) {
        if (colbase + j >= n) break;
        float bv[V];
#pragma unroll
        for (int v = 0; v < V; ++v) bv[v] = 0.f;
        fma_row<TB, V>(d, colbase + j, 1.f, c0, vec_ok, bv);
#pragma unroll
        for (int i = 0; i < RB; ++i) {
          if (i < rb) {
            float a = (float)blk[i * cb + j];
#pragma unroll
            for (int v = 0; v < V; ++v) acc[i][v] = fmaf(a, bv[v], acc[i][v]);
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < RB; ++i) {
      int64_t r = b * br + i;
      if (i < rb && r < m) store_row<V>(d, r, c0, false, acc[i]);
    }
  }
}

template <typename TB, int S>
void spmm_csr_merge(sfg_context* ctx, const sfg_tensor* a, const int32_t* col, const float* fv, Dense d) {
  const int64_t total = a->m + a->nnz;
  const int64_t nchunks = ceil_div(total, kMergeItems);
  // scratch: cuts[nchunks + 1] | carry rows[nchunks] | carry values[nchunks][nd]
  const size_t cut_b = ((size_t)(nchunks + 1) * sizeof(int2) + 15) & ~size_t(15);
  const size_t row_b = ((size_t)nchunks * 4 + 15) & ~size_t(15);
  const size_t val_b = (size_t)nchunks * d.nd * 4;
  char* s = static_cast<char*>(scratch(ctx, cut_b + row_b + val_b));
  auto* cuts = reinterpret_cast<int2*>(s);
  Carry cy{reinterpret_cast<int32_t*>(s + cut_b), reinterpret_cast<float*>(s + cut_b + row_b)};
  SFG_LAUNCH(k_merge_cuts, (int)std::min<int64_t>(ceil_div(nchunks + 1, 256), (int64_t)ctx->sms * 8), 256, 0,
             ctx->stream, a->ptr, a->m, a->nnz, nchunks + 1, cuts);
  const bool vec4 = d.ldb % 4 == 0 && d.ldc % 4 == 0 &&
                    ((reinterpret_cast<uintptr_t>(d.b) | reinterpret_cast<uintptr_t>(d.c)) & 15) == 0;
  auto grid_for = [&](int64_t warps_needed) {
    return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(warps_needed, kBlock / 32), (int64_t)ctx->sms * 16));
  };
  const int32_t m = (int32_t)a->m;
#define SFG_MERGE(G, V, U, VEC, ONE, MB, CC)                                                                      \
  SFG_LAUNCH((k_spmm_merge<TB, G, V, U, VEC, ONE, MB, S>), grid_for(nchunks * (CC)), kBlock, 0, ctx->stream, \
             a->ptr, col, fv, cuts, nchunks, m, d, cy)
  // nd = 32 on config 5 (SpMM ms): this unrolled step, 5 CTAs/SM 24.6;
  // 4 CTAs/SM 24.9; kU = 2 at 6 CTAs/SM 25.3; kU = 6 / 8 at 4 CTAs/SM 41.0 /
  // 43.8 (spills, code size); the row-end path as a rolled
  // loop (smaller code, more instructions) 26.3; the first version of this
  // kernel with the zeroing of empty rows inside every row close (code 5x
  // the size, instruction-cache bound) 44
  if (vec4 && d.nd == 32) SFG_MERGE(4, 4, 4, true, true, 5, 1);
  else if (vec4 && d.nd == 16) SFG_MERGE(8, 4, 4, true, true, 5, 1);
  else if (vec4 && d.nd == 64) SFG_MERGE(2, 4, 4, true, true, 5, 1);
  else if (vec4 && d.nd % 128 == 0) SFG_MERGE(1, 4, 4, true, false, 5, d.nd / 128);
  else SFG_MERGE(1, 1, 8, false, false, 5, ceil_div(d.nd, 32));
#undef SFG_MERGE
  carry_fix(ctx, cy.row, cy.val, nchunks, d.nd, d.c, d.ldc);
}

// BCSR / BELL with 128-column chunks of the dense operand (nd % 128 == 0,
// aligned B and C): register-tiled CUDA-core kernel for the shapes the
// tensor-core path does not take (fp32 values, 4x4 / 8x8 blocks). A warp
// owns (block row, 128 columns): lane l holds C[rows of the block row][4 l ..
// 4 l + 3] in registers (RB x 4 accumulators). Per block the warp stages the
// r x c value block in its shared-memory slot (fp32, row-major, padded to
// CB columns), then walks the block's columns four at a time: four B-row
// loads (16 bytes per lane) and, per block row r, one 16-byte shared load
// of a[r][j..j+3] broadcast to the warp and 16 FMAs. Per 16x16 block: 16
// B-row loads, 64 shared loads, 1,024 FMAs per lane.
template <typename TB, typename TA, int RB, int CB, bool kBell>
__global__ void __launch_bounds__(kBlock, RB == 16 ? 1 : 2) k_spmm_bcsr128(const int32_t* __restrict__ ptr,
                                                             const int32_t* __restrict__ bcol,
                                                             const TA* __restrict__ val, int64_t nbr, int32_t m,
                                                             int32_t n, int32_t br, int32_t bc, int32_t rb,
                                                             int32_t cb, Dense d, int64_t kslots) {
  static_assert(CB % 4 == 0 && RB <= 16 && CB <= 16, "block tile");
  __shared__ __align__(16) float s_blk[kBlock / 32][RB * CB];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  float* a_s = s_blk[wid];
  const int chunks = d.nd / 128;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int slots = rb * cb;
  for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nbr * chunks; w += warps) {
    const int64_t b = w / chunks;
    const int c0 = (int)(w - b * chunks) * 128 + lane * 4;
    float acc[RB][4];
#pragma unroll
    for (int i = 0; i < RB; ++i)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[i][v] = 0.f;
    const int64_t s = kBell ? 0 : __ldg(ptr + b), e = kBell ? kslots : __ldg(ptr + b + 1);
    for (int64_t kk = s; kk < e; ++kk) {
      const int64_t k = kBell ? kk * nbr + b : kk;
      const int colbase = __ldg(bcol + k) * bc;
      const TA* blk = val + k * slots;
      __syncwarp();
      for (int q = lane; q < RB * CB; q += 32) {
        const int i = q / CB, j = q - i * CB;
        a_s[q] = i < rb && j < cb ? (float)blk[i * cb + j] : 0.f;
      }
      __syncwarp();
#pragma unroll
      for (int j0 = 0; j0 < CB; j0 += 4) {
        float bv[4][4];
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const int col = colbase + j0 + jj;
          if (j0 + jj < cb && col < n) {
            BRow<TB>::template load<4>(static_cast<const TB*>(d.b) + (int64_t)col * d.ldb + c0, bv[jj]);
          } else {
#pragma unroll
            for (int v = 0; v < 4; ++v) bv[jj][v] = 0.f;
          }
        }
#pragma unroll
        for (int i = 0; i < RB; ++i) {
          const float4 a4 = *reinterpret_cast<const float4*>(a_s + i * CB + j0);
          const float av[4] = {a4.x, a4.y, a4.z, a4.w};
#pragma unroll
          for (int jj = 0; jj < 4; ++jj)
#pragma unroll
            for (int v = 0; v < 4; ++v) acc[i][v] = fmaf(av[jj], bv[jj][v], acc[i][v]);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < RB; ++i) {
      const int64_t r = b * br + i;
      if (i < rb && r < m) {
        float* crow = d.c + r * d.ldc + c0;
        float4 o = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
        if (d.acc) {
          const float4 p = *reinterpret_cast<const float4*>(crow);
          o.x += p.x, o.y += p.y, o.z += p.z, o.w += p.w;
        }
        *reinterpret_cast<float4*>(crow) = o;
      }
    }
  }
}

// The same product for exact tiles (r = RB, c = CB: 4x4, 8x8, 16x16 blocks)
// with the operands staged by cp.async in a two-deep ring per warp, so a
// warp keeps a whole stage of B rows in flight without holding them in
// registers (the B of config 4 is 268 MB in fp32, more than L2: its rows
// come from HBM and the kernel is bound by how many are in flight). A stage
// is 16 / CB blocks = 16 B-row slices of 512 bytes (fp32 B) plus the value
// blocks; the block columns of the stage after next are loaded a stage
// ahead, so issuing a stage never waits on them.
__device__ __forceinline__ void cp_async16_zfill(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async8_zfill(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(valid ? 8 : 0)
               : "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <typename TB, typename TA, int RB, int CB, bool kBell>
__global__ void __launch_bounds__(kBlock, 1) k_spmm_bcsr128p(const int32_t* __restrict__ ptr,
                                                              const int32_t* __restrict__ bcol,
                                                              const TA* __restrict__ val, int64_t nbr, int32_t m,
                                                              int32_t n, int32_t br, Dense d, int64_t kslots) {
  constexpr int kPer = 16 / CB;               // blocks per stage
  constexpr int kRows = 16;                   // B rows per stage
  constexpr int kBW = 4 * (int)sizeof(TB);    // B bytes per lane per row (4 columns)
  constexpr int kABytes = RB * CB * (int)sizeof(TA);
  constexpr int kAChunks = kABytes / 16;      // 16-byte pieces of one value block
  static_assert(kABytes % 16 == 0, "value blocks in 16-byte pieces");
  struct Stage {
    uint8_t b[kRows][32 * kBW];
    uint8_t a[kPer][kABytes];
  };
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  Stage* ring = reinterpret_cast<Stage*>(smem_raw) + wid * 2;
  const int chunks = d.nd / 128;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const TB* bbase = static_cast<const TB*>(d.b);
  for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nbr * chunks; w += warps) {
    const int64_t b = w / chunks;
    const int cw = (int)(w - b * chunks) * 128;
    const int c0 = cw + lane * 4;
    float acc[RB][4];
#pragma unroll
    for (int i = 0; i < RB; ++i)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[i][v] = 0.f;
    const int64_t s = kBell ? 0 : __ldg(ptr + b), e = kBell ? kslots : __ldg(ptr + b + 1);
    const int64_t nst = (e - s + kPer - 1) / kPer;
    auto blk_of = [&](int64_t kk) -> int64_t { return kBell ? kk * nbr + b : kk; };
    // block column of block kk (lane t < kPer holds block t of a stage)
    auto load_bcol = [&](int64_t st) -> int {
      const int64_t kk = s + st * kPer + lane;
      return lane < kPer && kk < e ? __ldg(bcol + blk_of(kk)) : -1;
    };
    auto issue = [&](int64_t st, int bc_lane) {
      Stage& g = ring[st & 1];
#pragma unroll
      for (int t = 0; t < kPer; ++t) {
        const int bcv = __shfl_sync(kFull, bc_lane, t);
        const int64_t kk = s + st * kPer + t;
#pragma unroll
        for (int j = 0; j < CB; ++j) {
          const int col = bcv * CB + j;
          const bool ok = bcv >= 0 && col < n;
          const TB* src = bbase + (ok ? (int64_t)col * d.ldb + c0 : 0);
          if constexpr (kBW == 16) cp_async16_zfill(&g.b[t * CB + j][lane * 16], src, ok);
          else cp_async8_zfill(&g.b[t * CB + j][lane * 8], src, ok);
        }
        const uint8_t* asrc = reinterpret_cast<const uint8_t*>(val + (bcv >= 0 ? blk_of(kk) : 0) * RB * CB);
        for (int q = lane; q < kAChunks; q += 32) cp_async16_zfill(&g.a[t][q * 16], asrc + q * 16, bcv >= 0);
      }
      cp_async_commit();
    };
    int bc_next = load_bcol(0);
    if (nst > 0) issue(0, bc_next);
    bc_next = load_bcol(1);
    for (int64_t st = 0; st < nst; ++st) {
      if (st + 1 < nst) issue(st + 1, bc_next);
      else cp_async_commit();  // keep the group count: wait_group 1 below
      bc_next = load_bcol(st + 2);
      cp_async_wait<1>();
      __syncwarp();
      const Stage& g = ring[st & 1];
#pragma unroll
      for (int t = 0; t < kPer; ++t) {
#pragma unroll
        for (int j0 = 0; j0 < CB; j0 += 4) {
          float bv[4][4];
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            const uint8_t* pb = &g.b[t * CB + j0 + jj][lane * kBW];
            if constexpr (kBW == 16) {
              const float4 q = *reinterpret_cast<const float4*>(pb);
              bv[jj][0] = q.x, bv[jj][1] = q.y, bv[jj][2] = q.z, bv[jj][3] = q.w;
            } else {
              const uint2 q = *reinterpret_cast<const uint2*>(pb);
              bv[jj][0] = __uint_as_float(q.x << 16), bv[jj][1] = __uint_as_float(q.x & 0xffff0000u);
              bv[jj][2] = __uint_as_float(q.y << 16), bv[jj][3] = __uint_as_float(q.y & 0xffff0000u);
            }
          }
#pragma unroll
          for (int i = 0; i < RB; ++i) {
            float av[4];
            if constexpr (sizeof(TA) == 4) {
              const float4 a4 = *reinterpret_cast<const float4*>(&g.a[t][(i * CB + j0) * 4]);
              av[0] = a4.x, av[1] = a4.y, av[2] = a4.z, av[3] = a4.w;
            } else {
              const uint2 q = *reinterpret_cast<const uint2*>(&g.a[t][(i * CB + j0) * 2]);
              av[0] = __uint_as_float(q.x << 16), av[1] = __uint_as_float(q.x & 0xffff0000u);
              av[2] = __uint_as_float(q.y << 16), av[3] = __uint_as_float(q.y & 0xffff0000u);
            }
#pragma unroll
            for (int jj = 0; jj < 4; ++jj)
#pragma unroll
              for (int v = 0; v < 4; ++v) acc[i][v] = fmaf(av[jj], bv[jj][v], acc[i][v]);
          }
        }
      }
      __syncwarp();  // the slot is refilled by the next iteration's issue
    }
    cp_async_wait<0>();
#pragma unroll
    for (int i = 0; i < RB; ++i) {
      const int64_t r = b * br + i;
      if (r < m) {
        float* crow = d.c + r * d.ldc + c0;
        float4 o = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
        if (d.acc) {
          const float4 p = *reinterpret_cast<const float4*>(crow);
          o.x += p.x, o.y += p.y, o.z += p.z, o.w += p.w;
        }
        *reinterpret_cast<float4*>(crow) = o;
      }
    }
  }
}

template <typename TB, int V>
void launch_fmt(sfg_context* ctx, const sfg_tensor* a, const Dense& d) {
  int64_t chunks = ceil_div(d.nd, 32 * V);
  auto grid_for = [&](int64_t warps_needed) {
    return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(warps_needed, kBlock / 32),
                                                      (int64_t)ctx->sms * 16));
  };
  const float* fv = static_cast<const float*>(a->val);
  const int64_t stored_rows = a->kind == SFG_DCSR ? tensor_nnr(a) : a->m;
  const bool short_rows = stored_rows > 0 && a->nnz <= 8 * stored_rows;  // <= 8 entries per row
  // measured on config 3 (3.6 M rows of ~2.3 entries, nd = 64), SpMM ms:
  // (R, kK) = (24, 8) 0.70, (31, 8) 0.71, (16, 8) 0.73, (16, 4) 0.79,
  // (8, 4) 0.83, (16, 16) 0.92
  constexpr int kBatchRows = 24, kBatchK = 8;
  switch (a->kind) {
    case SFG_CSR:
      if (a->m == 0) break;
      spmm_csr_merge<TB, 1>(ctx, a, a->idx, fv, d);
      break;
    case SFG_LIL: {
      if (a->m == 0) break;
      const auto* rec = static_cast<const int32_t*>(a->val);
      spmm_csr_merge<TB, 2>(ctx, a, rec, reinterpret_cast<const float*>(rec + 1), d);
      break;
    }
    case SFG_DCSR: {
      if (stored_rows == 0) break;
      const int32_t* rows = a->kind == SFG_DCSR ? a->row : nullptr;
      if (short_rows && d.nd % (32 * V) == 0 && d.ldb % V == 0 && d.ldc % V == 0 &&
          ((reinterpret_cast<uintptr_t>(d.b) | reinterpret_cast<uintptr_t>(d.c)) & (4 * V - 1)) == 0)
        SFG_LAUNCH((k_spmm_rows_batch<TB, V, kBatchRows, kBatchK, true>),
                   grid_for(ceil_div(stored_rows, kBatchRows) * chunks), kBlock, 0, ctx->stream, rows, a->ptr,
                   a->idx, fv, stored_rows, d);
      else if (short_rows)
        SFG_LAUNCH((k_spmm_rows_batch<TB, V, kBatchRows, kBatchK, false>),
                   grid_for(ceil_div(stored_rows, kBatchRows) * chunks), kBlock, 0, ctx->stream, rows, a->ptr,
                   a->idx, fv, stored_rows, d);
      else
        SFG_LAUNCH((k_spmm_rows<TB, V>), grid_for(stored_rows * chunks), kBlock, 0, ctx->stream, rows,
                   a->ptr, a->idx, fv, stored_rows, d);
      break;
    }
    case SFG_ELL:
      SFG_LAUNCH((k_spmm_ell<TB, V>), grid_for(a->m * chunks), kBlock, 0, ctx->stream, a->idx, fv,
                 (int32_t)a->m, (int32_t)a->k, d);
      break;
    case SFG_BDIA:
      if (a->m)
        SFG_LAUNCH((k_spmm_bdia<TB, V>), grid_for(a->m * chunks), kBlock, 0, ctx->stream, a->ptr, a->idx, fv, a->m,
                   a->n, (int32_t)a->br, (int32_t)a->rb, d);
      break;
    case SFG_DIA:
    case SFG_DIAV:
      if (a->m)
        SFG_LAUNCH((k_spmm_dia<TB, V>), grid_for(a->m * chunks), kBlock, 0, ctx->stream, a->slots, fv, a->m, a->n,
                   a->k, a->kind == SFG_DIAV, d);
      break;
    case SFG_COO:
    case SFG_DOK:
      if (a->nnz) {
        const int64_t nq = ceil_div(a->nnz, 32 * kCooIters);
        const size_t row_b = ((size_t)nq * 4 + 15) & ~size_t(15);
        char* s = static_cast<char*>(scratch(ctx, row_b + (size_t)nq * d.nd * 4));
        Carry cy{reinterpret_cast<int32_t*>(s), reinterpret_cast<float*>(s + row_b)};
        if (a->kind == SFG_DOK) {  // records {row, col, val}
          const auto* rec = static_cast<const int32_t*>(a->val);
          SFG_LAUNCH((k_spmm_coo<TB, V, 3>), grid_for(nq * chunks), kBlock, 0, ctx->stream, rec, rec + 1,
                     reinterpret_cast<const float*>(rec + 2), a->nnz, d, cy);
        } else {
          SFG_LAUNCH((k_spmm_coo<TB, V, 1>), grid_for(nq * chunks), kBlock, 0, ctx->stream, a->row, a->idx, fv,
                     a->nnz, d, cy);
        }
        carry_fix(ctx, cy.row, cy.val, nq, d.nd, d.c, d.ldc);
      }
      break;
    case SFG_CSC:
      if (a->nnz)
        SFG_LAUNCH((k_spmm_csc<TB, V>), grid_for(a->n * chunks), kBlock, 0, ctx->stream, a->ptr,
                   a->idx, fv, (int32_t)a->n, d);
      break;
    case SFG_BCSR:
    case SFG_BELL: {
      if (a->nbr == 0 || a->nnz == 0) break;
      if (a->rb > 16) raise(SFG_ERR_INVALID_OPERATION, "BCSR SpMM: block rows > 16 not supported");
      const bool v128 = d.nd % 128 == 0 && d.ldb % 4 == 0 && d.ldc % 4 == 0 && a->cb <= 16 &&
                        ((reinterpret_cast<uintptr_t>(d.b) | reinterpret_cast<uintptr_t>(d.c)) & 15) == 0;
      if (v128) {
        // register-tiled path (fp32 or bf16 values; the 16x16 bf16 / bf16-B
        // case with nd = 128 went to the tensor cores above)
        const int g128 = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(a->nbr * (d.nd / 128), kBlock / 32),
                                                                     (int64_t)ctx->sms * 16));
        const bool bell = a->kind == SFG_BELL, bf = a->dtype == SFG_BF16;
        const int cbt = a->cb <= 4 ? 4 : a->cb <= 8 ? 8 : 16;
        const int rbt = a->rb <= 4 ? 4 : a->rb <= 8 ? 8 : 16;
        if (a->rb == a->cb && a->rb == rbt && a->cb == cbt) {
          // exact square tiles: the cp.async-staged kernel (8 warps, two
          // stages each, one CTA per SM)
          auto go = [&](auto kern, size_t stage_bytes, auto v) {
            const size_t smem = (size_t)(kBlock / 32) * 2 * stage_bytes;
            SFG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            const int gp = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(a->nbr * (d.nd / 128), kBlock / 32),
                                                                       (int64_t)ctx->sms));
            SFG_LAUNCH(kern, gp, kBlock, smem, ctx->stream, a->ptr, a->idx, v, a->nbr,
                       (int)a->m, (int)a->n, (int)a->br, d, a->k);
          };
#define SFG_B128P(T, TAT)                                                                                          \
  if (rbt == T) {                                                                                                   \
    constexpr size_t kSB = 16 * 32 * 4 * sizeof(TB) + (16 / T) * T * T * sizeof(TAT);                             \
    if (bell)                                                                                                       \
      go(k_spmm_bcsr128p<TB, TAT, T, T, true>, kSB, static_cast<const TAT*>(a->val));                              \
    else                                                                                                            \
      go(k_spmm_bcsr128p<TB, TAT, T, T, false>, kSB, static_cast<const TAT*>(a->val));                             \
    break;                                                                                                          \
  }
          if (bf && !bell) {
            SFG_B128P(4, __nv_bfloat16) SFG_B128P(8, __nv_bfloat16) SFG_B128P(16, __nv_bfloat16)
          } else {
            SFG_B128P(4, float) SFG_B128P(8, float) SFG_B128P(16, float)
          }
#undef SFG_B128P
        }
#define SFG_B128(RBT, CBT)                                                                                      \
  if (rbt == RBT && cbt == CBT) {                                                                               \
    if (bell)                                                                                                   \
      SFG_LAUNCH((k_spmm_bcsr128<TB, float, RBT, CBT, true>), g128, kBlock, 0, ctx->stream, a->ptr, a->idx, fv,  \
                 a->nbr, (int)a->m, (int)a->n, (int)a->br, (int)a->bc, (int)a->rb, (int)a->cb, d, a->k);        \
    else if (bf)                                                                                                \
      SFG_LAUNCH((k_spmm_bcsr128<TB, __nv_bfloat16, RBT, CBT, false>), g128, kBlock, 0, ctx->stream, a->ptr,     \
                 a->idx, static_cast<const __nv_bfloat16*>(a->val), a->nbr, (int)a->m, (int)a->n, (int)a->br,   \
                 (int)a->bc, (int)a->rb, (int)a->cb, d, a->k);                                                 \
    else                                                                                                        \
      SFG_LAUNCH((k_spmm_bcsr128<TB, float, RBT, CBT, false>), g128, kBlock, 0, ctx->stream, a->ptr, a->idx, fv, \
                 a->nbr, (int)a->m, (int)a->n, (int)a->br, (int)a->bc, (int)a->rb, (int)a->cb, d, a->k);        \
    break;                                                                                                      \
  }
        SFG_B128(4, 4) SFG_B128(4, 8) SFG_B128(4, 16) SFG_B128(8, 4) SFG_B128(8, 8) SFG_B128(8, 16)
        SFG_B128(16, 4) SFG_B128(16, 8) SFG_B128(16, 16)
#undef SFG_B128
      }
      int g = grid_for(a->nbr * chunks);
#define SFG_BCSR_CASE(RB)                                                                                 \
  if (a->kind == SFG_BELL)                                                                                \
    SFG_LAUNCH((k_spmm_bcsr<TB, float, V, RB, true>), g, kBlock, 0, ctx->stream, a->ptr, a->idx, fv, a->nbr, \
               (int)a->m, (int)a->n, (int)a->br, (int)a->bc, (int)a->rb, (int)a->cb, d, a->k);            \
  else if (a->dtype == SFG_BF16)                                                                          \
    SFG_LAUNCH((k_spmm_bcsr<TB, __nv_bfloat16, V, RB, false>), g, kBlock, 0, ctx->stream, a->ptr, a->idx,  \
               static_cast<const __nv_bfloat16*>(a->val), a->nbr, (int)a->m, (int)a->n,                  \
               (int)a->br, (int)a->bc, (int)a->rb, (int)a->cb, d, a->k);                                  \
  else                                                                                                    \
    SFG_LAUNCH((k_spmm_bcsr<TB, float, V, RB, false>), g, kBlock, 0, ctx->stream, a->ptr, a->idx, fv,      \
               a->nbr, (int)a->m, (int)a->n, (int)a->br, (int)a->bc, (int)a->rb, (int)a->cb, d, a->k);
      if (a->rb <= 4) { SFG_BCSR_CASE(4) }
      else if (a->rb <= 8) { SFG_BCSR_CASE(8) }
      else { SFG_BCSR_CASE(16) }
#undef SFG_BCSR_CASE
      break;
    }
    default: raise(SFG_ERR_INVALID_OPERATION, "spmm: unsupported format");
  }
}

template <typename TB>
void launch_v(sfg_context* ctx, const sfg_tensor* a, const Dense& d) {
  // vector B loads need a B pointer aligned to the vector (callers may pass
  // any element offset)
  const uintptr_t pb = reinterpret_cast<uintptr_t>(d.b);
  if (d.nd >= 128 && pb % (4 * sizeof(TB)) == 0) launch_fmt<TB, 4>(ctx, a, d);
  else if (d.nd >= 64 && pb % (2 * sizeof(TB)) == 0) launch_fmt<TB, 2>(ctx, a, d);
  else launch_fmt<TB, 1>(ctx, a, d);
}

}  // namespace

namespace {
// One level of the carry reduction: a warp per group of 32 consecutive
// carry slots. Rows with carries form runs of consecutive slots (a row
// longer than a chunk); the warp walks its slots in order, lanes over the
// columns, the group's values loaded up front. A run ending inside the
// group is complete: its sum is added to C. The group is that row's only
// writer at this level and the levels run in order, so the add is an
// atomic only to make it a fire-and-forget reduction (a load-add-store
// would stall the warp once per run); the result does not depend on
// timing. The run still open at the group's end (the next slot carries the
// same row) becomes the group's carry for the next level, which sees 32x
// fewer slots.
__device__ __forceinline__ void carry_group(const int32_t* __restrict__ in_row, const float* __restrict__ in_val,
                                            int64_t n, int nd, float* __restrict__ c, int64_t ldc,
                                            int32_t* __restrict__ out_row, float* __restrict__ out_val, int64_t g) {
  const int lane = threadIdx.x & 31;
  const int64_t t0 = g * 32;
  const int cnt = (int)(n - t0 < 32 ? n - t0 : 32);
  const int rl = lane < cnt ? in_row[t0 + lane] : -1;
  const int next = t0 + 32 < n ? in_row[t0 + 32] : -1;
  const int last = __shfl_sync(kFull, rl, cnt - 1);
  const bool open = last >= 0 && last == next;
  if (nd == 1) {
    // one value per slot: lane t holds slot t; a head-flag segmented scan
    // (fixed shuffle order) sums each run, its last lane adds it
    float t = rl >= 0 ? in_val[t0 + lane] : 0.f;
    const int up = __shfl_up_sync(kFull, rl, 1);
    const unsigned heads = __ballot_sync(kFull, lane == 0 || up != rl);
    const int start = 31 - __clz(heads & (0xffffffffu >> (31 - lane)));
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const float u = __shfl_up_sync(kFull, t, o);
      if (lane - o >= start) t += u;
    }
    const int dn = __shfl_down_sync(kFull, rl, 1);
    const bool tail = lane == 31 || dn != rl;  // last slot of its run in this group
    if (tail && rl >= 0) {
      if (open && lane == cnt - 1) out_val[g] = t;
      else atomicAdd(c + (int64_t)rl * ldc, t);
    }
  } else {
    for (int cb = 0; cb < nd; cb += 32) {
      const int col = cb + lane;
      float acc = 0.f;
      int cur = -1;
      for (int t8 = 0; t8 < cnt; t8 += 8) {
        float vv[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int r = __shfl_sync(kFull, rl, (t8 + k) & 31);
          vv[k] = t8 + k < cnt && r >= 0 && col < nd ? in_val[(t0 + t8 + k) * nd + col] : 0.f;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int r = __shfl_sync(kFull, rl, (t8 + k) & 31);
          if (t8 + k < cnt && r >= 0 && r != cur) {
            if (cur >= 0 && col < nd) atomicAdd(c + (int64_t)cur * ldc + col, acc);
            cur = r;
            acc = 0.f;
          }
          acc += vv[k];
        }
      }
      if (cur >= 0 && col < nd) {
        if (open) out_val[g * nd + col] = acc;
        else atomicAdd(c + (int64_t)cur * ldc + col, acc);
      }
    }
  }
  if (lane == 0) out_row[g] = open ? last : -1;
}

__global__ void __launch_bounds__(256) k_carry_level(const int32_t* __restrict__ in_row,
                                                     const float* __restrict__ in_val, int64_t n, int nd,
                                                     float* __restrict__ c, int64_t ldc,
                                                     int32_t* __restrict__ out_row, float* __restrict__ out_val) {
  const int64_t groups = (n + 31) / 32;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; g < groups; g += warps)
    carry_group(in_row, in_val, n, nd, c, ldc, out_row, out_val, g);
}

// The last level: a warp per slot; the first slot of each run adds the
// run's carries, in slot order, to C. Runs are short here (a row spanning
// r chunks leaves a run of r / 32^levels slots).
__global__ void __launch_bounds__(256) k_carry_runs(const int32_t* __restrict__ in_row,
                                                    const float* __restrict__ in_val, int64_t n, int nd,
                                                    float* __restrict__ c, int64_t ldc) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < n; q += warps) {
    const int r = in_row[q];
    if (r < 0 || (q > 0 && in_row[q - 1] == r)) continue;
    int64_t t1 = q + 1;
    while (t1 < n && in_row[t1] == r) ++t1;
    for (int col = lane; col < nd; col += 32) {
      float acc = 0.f;
      for (int64_t t = q; t < t1; ++t) acc += in_val[t * nd + col];
      atomicAdd(c + (int64_t)r * ldc + col, acc);
    }
  }
}
}  // namespace

void carry_fix(sfg_context* ctx, const int32_t* row, const float* val, int64_t n, int nd, float* c, int64_t ldc) {
  if (n <= 0) return;
  const int64_t n2 = (n + 31) / 32;
  int32_t* rows[2] = {nullptr, nullptr};
  float* vals[2] = {nullptr, nullptr};
  if (n > 1024) {
    rows[0] = dalloc_n<int32_t>(ctx, n2);
    rows[1] = dalloc_n<int32_t>(ctx, n2);
    vals[0] = dalloc_n<float>(ctx, n2 * nd);
    vals[1] = dalloc_n<float>(ctx, n2 * nd);
  }
  const int32_t* ir = row;
  const float* iv = val;
  int lvl = 0;
  while (n > 1024) {  // 32 slots to one per level
    const int64_t groups = (n + 31) / 32;
    const int grid = (int)std::min<int64_t>(ceil_div(groups, 8), (int64_t)ctx->sms * 16);
    SFG_LAUNCH(k_carry_level, grid, 256, 0, ctx->stream, ir, iv, n, nd, c, ldc, rows[lvl & 1], vals[lvl & 1]);
    ir = rows[lvl & 1];
    iv = vals[lvl & 1];
    n = groups;
    ++lvl;
  }
  SFG_LAUNCH(k_carry_runs, (int)std::max<int64_t>(1, ceil_div(n, 8)), 256, 0, ctx->stream, ir, iv, n, nd, c, ldc);
  for (int k = 0; k < 2; ++k) {
    if (rows[k]) dfree(ctx, rows[k]);
    if (vals[k]) dfree(ctx, vals[k]);
  }
}

// Tensor-core BCSR path (bcsr_tc.cu); returns false when not applicable.
bool spmm_bcsr_tc(sfg_context* ctx, const sfg_tensor* a, const void* b, int b_dtype, int64_t nd,
                  int64_t ldb, float* c, int64_t ldc, bool accumulate);

void spmm(sfg_context* ctx, const sfg_tensor* a, const void* b, int b_dtype, int64_t nd,
          int64_t ldb, float* c, int64_t ldc, bool accumulate) {
  if (a->kind == SFG_HYB || a->kind == SFG_HBELL) {
    spmm(ctx, a->part[0], b, b_dtype, nd, ldb, c, ldc, accumulate);
    spmm(ctx, a->part[1], b, b_dtype, nd, ldb, c, ldc, true);
    return;
  }
  if (a->kind == SFG_BCSR && spmm_bcsr_tc(ctx, a, b, b_dtype, nd, ldb, c, ldc, accumulate)) return;
  if (a->kind == SFG_CSB || a->kind == SFG_C2SR || a->kind == SFG_DCSC || a->kind == SFG_CISR ||
      a->kind == SFG_CISRP) {  // the entries back in row order, then COO
    sfg_tensor* coo = a->kind == SFG_CSB    ? csb_to_coo(ctx, a)
                      : a->kind == SFG_C2SR ? c2sr_to_coo(ctx, a)
                      : a->kind == SFG_DCSC ? dcsc_to_coo(ctx, a)
                                            : cisr_to_coo(ctx, a);
    try {
      spmm(ctx, coo, b, b_dtype, nd, ldb, c, ldc, accumulate);
    } catch (...) {
      free_tensor_arrays(coo);
      delete coo;
      throw;
    }
    free_tensor_arrays(coo);
    delete coo;
    return;
  }
  if (a->kind == SFG_DCSR && !accumulate && a->m > 0) {
    if (tensor_nnr(a) == 0) {
      if (ldc == nd) SFG_CUDA(cudaMemsetAsync(c, 0, a->m * ldc * sizeof(float), ctx->stream));
      else SFG_CUDA(cudaMemset2DAsync(c, ldc * sizeof(float), 0, nd * sizeof(float), a->m, ctx->stream));
      return;
    }
    // stored rows are written whole by the kernel, which also zeroes the
    // gaps between them
    Dense d{b, ldb, c, ldc, (int32_t)nd, 0, 0, a->m};
    if (b_dtype == SFG_BF16) launch_v<__nv_bfloat16>(ctx, a, d);
    else launch_v<float>(ctx, a, d);
    return;
  }
  bool zero_first =
      !accumulate && (a->kind == SFG_COO || a->kind == SFG_DOK || a->kind == SFG_CSC || a->kind == SFG_BCSR ||
                      a->kind == SFG_BELL);
  if (zero_first && a->m > 0) {
    if (ldc == nd)
      SFG_CUDA(cudaMemsetAsync(c, 0, a->m * ldc * sizeof(float), ctx->stream));
    else
      SFG_CUDA(cudaMemset2DAsync(c, ldc * sizeof(float), 0, nd * sizeof(float), a->m, ctx->stream));
  }
  // kernels that own whole rows write with accumulate semantics after zeroing
  Dense d{b, ldb, c, ldc, (int32_t)nd, (accumulate || zero_first) ? 1 : 0, accumulate ? 1 : 0};
  if (b_dtype == SFG_BF16) launch_v<__nv_bfloat16>(ctx, a, d);
  else launch_v<float>(ctx, a, d);
}

}  // namespace sfg
