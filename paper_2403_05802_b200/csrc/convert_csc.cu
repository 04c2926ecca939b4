// convert_csc.cu — COO -> CSC.
//
// Reference: plan Swap(0,1) Sort Fill(0) Merge(0) (
// operators.hpp:234-241 Swap, 298-301 Sort = stable sort_entries,
// tensor.hpp:98-114). The result is uniquely determined: column pointers
// ptr[n+1], and within each column the rows in ascending order (the input
// is row-sorted and the sort is stable), materialized like CSR with the
// roles of rows and columns exchanged (storage.hpp:171-200).
//
// Device plan. Fast path (every column holds <= kShortCol entries, e.g. the
// hypersparse config 3): column histogram (RED atomics) -> single-pass
// look-back scan -> atomic-cursor scatter -> per-column insertion sort by
// row, which restores the stable order. Any longer column switches to the
// general path: stable LSD radix sort on the column bits with the row
// carried in the upper key half, then compression of the sorted columns.
#include "async.cuh"
#include "devutil.cuh"
#include "internal.cuh"

namespace sfg {

namespace {

constexpr int kBlock = 256;
constexpr int kShortCol = 32;

__global__ void __launch_bounds__(kBlock) k_col_hist(const int32_t* __restrict__ col, int64_t nnz,
                                                      int32_t* __restrict__ cnt) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(cnt + ld_stream(col + e), 1);
}

// Exclusive scan of counts -> ptr[0..n] and a cursor copy; max count.
constexpr int kItems = 16;
constexpr int kTile = kBlock * kItems;

__global__ void __launch_bounds__(kBlock) k_count_scan(const int32_t* __restrict__ cnt, int32_t n,
                                                        int32_t* __restrict__ ptr, int32_t* __restrict__ cursor,
                                                        unsigned long long* __restrict__ status,
                                                        uint32_t epoch, int32_t* __restrict__ maxcnt) {
  __shared__ uint32_t smem[34];
  __shared__ uint32_t slot;
  const int64_t c0 = (int64_t)blockIdx.x * kTile + (int64_t)threadIdx.x * kItems;
  const bool full = c0 + kItems <= n;  // 16-byte vector loads / stores
  uint32_t v[kItems];
  uint32_t sum = 0;
  int32_t mx = 0;
  if (full) {
#pragma unroll
    for (int q = 0; q < kItems / 4; ++q) {
      const int4 w = __ldg(reinterpret_cast<const int4*>(cnt + c0) + q);
      v[4 * q] = w.x, v[4 * q + 1] = w.y, v[4 * q + 2] = w.z, v[4 * q + 3] = w.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < kItems; ++i) v[i] = c0 + i < n ? (uint32_t)__ldg(cnt + c0 + i) : 0u;
  }
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    sum += v[i];
    mx = max(mx, (int32_t)v[i]);
  }
  uint32_t total;
  uint32_t excl = block_exclusive_scan<uint32_t, kBlock>(sum, smem, &total);
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0) atomicMax(maxcnt, mx);
  uint32_t p = lookback_prefix(status, epoch, blockIdx.x, total, &slot) + excl;
  if (full) {
#pragma unroll
    for (int q = 0; q < kItems / 4; ++q) {
      int4 w;
      w.x = (int32_t)p, p += v[4 * q];
      w.y = (int32_t)p, p += v[4 * q + 1];
      w.z = (int32_t)p, p += v[4 * q + 2];
      w.w = (int32_t)p, p += v[4 * q + 3];
      reinterpret_cast<int4*>(ptr + c0)[q] = w;
      reinterpret_cast<int4*>(cursor + c0)[q] = w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      if (c0 + i < n) {
        ptr[c0 + i] = (int32_t)p;
        cursor[c0 + i] = (int32_t)p;
        p += v[i];
      }
    }
  }
  if (c0 + kItems >= n && c0 < n) ptr[n] = (int32_t)p;
}

// Atomic-cursor scatter; the order inside a column is fixed afterwards
// (mostly ascending already: earlier entries tend to claim earlier slots).
// kScatterU entries per thread are in flight at once (the atomic's round
// trip dominates).
constexpr int kScatterU = 4;

__global__ void __launch_bounds__(kBlock) k_csc_scatter(const int32_t* __restrict__ row,
                                                         const int32_t* __restrict__ col,
                                                         const float* __restrict__ val, int64_t nnz,
                                                         int32_t* __restrict__ cursor,
                                                         int32_t* __restrict__ orow,
                                                         float* __restrict__ oval) {
  // the scattered 4-byte stores fill their lines over the whole pass: keep
  // those lines (and k_csc_fix's re-read) in L2 ahead of the streamed input
  const uint64_t once = l2_evict_first(), keep = l2_evict_last();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += kScatterU * stride) {
    int c[kScatterU], pos[kScatterU];
#pragma unroll
    for (int u = 0; u < kScatterU; ++u) c[u] = e + u * stride < nnz ? (int)ld_hint(col + e + u * stride, once) : -1;
#pragma unroll
    for (int u = 0; u < kScatterU; ++u)
      if (c[u] >= 0) pos[u] = atomicAdd(cursor + c[u], 1);
#pragma unroll
    for (int u = 0; u < kScatterU; ++u)
      if (c[u] >= 0) {
        st_hint(orow + pos[u], ld_hint(row + e + u * stride, once), keep);
        st_hint(oval + pos[u], ld_hint(val + e + u * stride, once), keep);
      }
  }
}

// Columns are short here (<= kShortCol): per-thread insertion sort by row.
__global__ void __launch_bounds__(kBlock) k_csc_fix(const int32_t* __restrict__ ptr, int32_t n,
                                                     int32_t* __restrict__ orow,
                                                     float* __restrict__ oval) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n;
       c += (int64_t)gridDim.x * blockDim.x) {
    int s = __ldg(ptr + c), e = __ldg(ptr + c + 1);
    if (e - s < 2) continue;
    for (int i = s + 1; i < e; ++i) {
      int r = orow[i];
      float v = oval[i];
      int j = i - 1;
      while (j >= s && orow[j] > r) {
        orow[j + 1] = orow[j];
        oval[j + 1] = oval[j];
        --j;
      }
      orow[j + 1] = r;
      oval[j + 1] = v;
    }
  }
}

// General path: key = row << 32 | col, payload = value bits.
__global__ void __launch_bounds__(kBlock) k_csc_keys(const int32_t* __restrict__ row,
                                                      const int32_t* __restrict__ col,
                                                      const float* __restrict__ val, int64_t nnz,
                                                      uint64_t* __restrict__ keys,
                                                      uint32_t* __restrict__ pay) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    keys[e] = ((uint64_t)(uint32_t)ld_stream(row + e) << 32) | (uint32_t)ld_stream(col + e);
    pay[e] = __float_as_uint(ld_stream(val + e));
  }
}

__global__ void __launch_bounds__(kBlock) k_csc_unpack(const uint64_t* __restrict__ keys,
                                                        const uint32_t* __restrict__ pay,
                                                        int64_t nnz, int32_t* __restrict__ ccol,
                                                        int32_t* __restrict__ crow,
                                                        float* __restrict__ cval) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k = keys[e];
    ccol[e] = (int32_t)(uint32_t)k;
    crow[e] = (int32_t)(k >> 32);
    cval[e] = __uint_as_float(pay[e]);
  }
}

int bits_for(int64_t extent) {
  int b = 0;
  while ((int64_t(1) << b) < extent) ++b;
  return b;
}

}  // namespace

sfg_tensor* coo_to_csc(sfg_context* ctx, const sfg_tensor* s) {
  const int64_t n = s->n, nnz = s->nnz;
  sfg_tensor* t = new_tensor(ctx, SFG_CSC, s->m, n);
  t->nnz = nnz;
  t->ptr = dalloc_n<int32_t>(ctx, n + 1);
  t->idx = dalloc_n<int32_t>(ctx, nnz);
  t->val = dalloc_n<float>(ctx, nnz);
  const float* sv = static_cast<const float*>(s->val);
  float* tv = static_cast<float*>(t->val);
  if (nnz == 0) {
    SFG_CUDA(cudaMemsetAsync(t->ptr, 0, (n + 1) * sizeof(int32_t), ctx->stream));
    return t;
  }
  int32_t* cnt = dalloc_n<int32_t>(ctx, n);
  int32_t* cursor = dalloc_n<int32_t>(ctx, n);
  int tiles = (int)ceil_div(n, kTile);
  auto* status = lookback_status(ctx, tiles);
  auto* maxcnt = static_cast<int32_t*>(scratch(ctx, 64));
  SFG_CUDA(cudaMemsetAsync(cnt, 0, n * sizeof(int32_t), ctx->stream));
  SFG_CUDA(cudaMemsetAsync(maxcnt, 0, sizeof(int32_t), ctx->stream));
  SFG_LAUNCH(k_col_hist, stream_grid(ctx, nnz, kBlock, 4), kBlock, 0, ctx->stream, s->idx, nnz, cnt);
  SFG_LAUNCH(k_count_scan, tiles, kBlock, 0, ctx->stream, cnt, (int32_t)n, t->ptr, cursor, status,
             ctx->epoch++, maxcnt);
  int32_t mx = 0;
  read_back(ctx, maxcnt, sizeof mx, &mx);
  if (mx <= kShortCol) {
    SFG_LAUNCH(k_csc_scatter, stream_grid(ctx, ceil_div(nnz, kScatterU), kBlock, 1), kBlock, 0, ctx->stream,
               s->row, s->idx, sv, nnz, cursor, t->idx, tv);
    SFG_LAUNCH(k_csc_fix, stream_grid(ctx, n, kBlock, 2), kBlock, 0, ctx->stream, t->ptr,
               (int32_t)n, t->idx, tv);
    dfree(ctx, cnt);
    dfree(ctx, cursor);
    return t;
  }
  dfree(ctx, cnt);
  dfree(ctx, cursor);
  // general path: stable radix sort on the column bits
  uint64_t* keys = dalloc_n<uint64_t>(ctx, nnz);
  uint32_t* pay = dalloc_n<uint32_t>(ctx, nnz);
  SFG_LAUNCH(k_csc_keys, stream_grid(ctx, nnz, kBlock, 4), kBlock, 0, ctx->stream, s->row, s->idx,
             sv, nnz, keys, pay);
  uint64_t *kres, *kalt;
  uint32_t *pres, *palt;
  radix_sort(ctx, keys, pay, nnz, bits_for(n), &kres, &pres, &kalt, &palt);
  int32_t* ccol = dalloc_n<int32_t>(ctx, nnz);
  int32_t* crow = dalloc_n<int32_t>(ctx, nnz);
  float* cval = dalloc_n<float>(ctx, nnz);
  SFG_LAUNCH(k_csc_unpack, stream_grid(ctx, nnz, kBlock, 4), kBlock, 0, ctx->stream, kres, pres, nnz,
             ccol, crow, cval);
  compress_sorted(ctx, ccol, crow, cval, nnz, n, t->ptr, t->idx, tv);
  for (void* p : {(void*)keys, (void*)pay, (void*)kalt, (void*)palt, (void*)ccol, (void*)crow,
                  (void*)cval})
    dfree(ctx, p);
  return t;
}

}  // namespace sfg
