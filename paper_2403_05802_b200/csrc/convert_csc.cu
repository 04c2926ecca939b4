// convert_csc.cu — COO -> CSC.
//
// Reference: plan Swap(0,1) Sort Fill(0) Merge(0) (
// operators.hpp:234-241 Swap, 298-301 Sort = stable sort_entries,
// tensor.hpp:98-114). The result is uniquely determined: column pointers
// ptr[n+1], and within each column the rows in ascending order (the input
// is row-sorted and the sort is stable), materialized like CSR with the
// roles of rows and columns exchanged (storage.hpp:171-200).
//
// Device plan. (1) Column-block partition (every block of 1,024 columns
// holds <= 4,096 entries, e.g. the hypersparse config 3): count per block,
// scan, scatter into block regions, sort each block in shared memory —
// below. (2) Otherwise, when every column holds <= kShortCol entries:
// column histogram (RED atomics) -> single-pass look-back scan ->
// atomic-cursor scatter -> per-column insertion sort by row, which restores
// the stable order. (3) Any longer column: stable LSD radix sort on the
// column bits with the row carried in the upper key half, then compression
// of the sorted columns. Config 3 (8.4 M entries, 4 M columns): (1) 0.35 ms,
// (2) 0.37 ms.
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

// ---------------------------------------------- column-block partition path
// Atomic-free in global memory and coalesced: (1) each of P CTAs counts its
// contiguous share of the entries per column block of kBlkCols columns (in
// shared memory); (2) an exclusive scan over (block, CTA) gives every CTA
// its write range inside every block's region; (3) the CTAs scatter their
// entries into those ranges (shared-memory cursors); (4) one CTA per column
// block loads its <= kBlkCap entries, counts them per column in shared
// memory, places them by column, insertion-sorts each (short) column by row
// and writes idx / val / ptr for its columns with coalesced stores.
constexpr int kBlkColBits = 10;
constexpr int kBlkCols = 1 << kBlkColBits;  // columns per block
constexpr int kBlkCap = 4096;               // entries one block CTA sorts in shared memory
constexpr int kMaxBlks = 8192;              // shared-memory counters of steps 1 and 3
constexpr int kPartCtas = 296;              // P (2 per SM)

__global__ void __launch_bounds__(kBlock) k_blk_count(const int32_t* __restrict__ col, int64_t nnz, int nb,
                                                       int32_t* __restrict__ counts) {
  __shared__ int32_t h[kMaxBlks];
  for (int i = threadIdx.x; i < nb; i += kBlock) h[i] = 0;
  __syncthreads();
  const int64_t per = (nnz + gridDim.x - 1) / gridDim.x;
  const int64_t e0 = blockIdx.x * per, e1 = min(nnz, e0 + per);
  for (int64_t e = e0 + threadIdx.x; e < e1; e += kBlock) atomicAdd(&h[ld_stream(col + e) >> kBlkColBits], 1);
  __syncthreads();
  for (int b = threadIdx.x; b < nb; b += kBlock) counts[(int64_t)b * gridDim.x + blockIdx.x] = h[b];
}

__global__ void __launch_bounds__(kBlock) k_blk_max(const int32_t* __restrict__ off, int nb, int p,
                                                     int32_t* __restrict__ mx) {
  int m = 0;
  for (int b = blockIdx.x * kBlock + threadIdx.x; b < nb; b += gridDim.x * kBlock)
    m = max(m, off[(int64_t)(b + 1) * p] - off[(int64_t)b * p]);
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) atomicMax(mx, m);
}

// Entries travel as (row << kBlkColBits | column within the block, value):
// rows must fit 32 - kBlkColBits bits (checked by the caller).
__global__ void __launch_bounds__(kBlock) k_blk_scatter(const int32_t* __restrict__ row,
                                                         const int32_t* __restrict__ col,
                                                         const float* __restrict__ val, int64_t nnz, int nb,
                                                         const int32_t* __restrict__ off,
                                                         uint32_t* __restrict__ tkey, float* __restrict__ tval) {
  __shared__ int32_t cur[kMaxBlks];
  for (int b = threadIdx.x; b < nb; b += kBlock) cur[b] = off[(int64_t)b * gridDim.x + blockIdx.x];
  __syncthreads();
  // the scattered stores fill their lines over the whole pass: keep them in
  // L2 (k_blk_sort reads them next) ahead of the streamed input
  const uint64_t once = l2_evict_first(), keep = l2_evict_last();
  const int64_t per = (nnz + gridDim.x - 1) / gridDim.x;
  const int64_t e0 = blockIdx.x * per, e1 = min(nnz, e0 + per);
  constexpr int U = 4;  // entries per thread in flight
  for (int64_t e = e0 + threadIdx.x; e < e1; e += U * kBlock) {
    uint32_t c[U], r[U], v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (e + u * kBlock < e1) {
        c[u] = ld_hint(col + e + u * kBlock, once);
        r[u] = ld_hint(row + e + u * kBlock, once);
        v[u] = ld_hint(val + e + u * kBlock, once);
      }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (e + u * kBlock < e1) {
        const int slot = atomicAdd(&cur[c[u] >> kBlkColBits], 1);
        st_hint(tkey + slot, (r[u] << kBlkColBits) | (c[u] & (kBlkCols - 1)), keep);
        st_hint(tval + slot, v[u], keep);
      }
  }
}

constexpr int kSortThreads = 512;

#ifndef SFG_BLKSORT_MINB
#define SFG_BLKSORT_MINB 1  // 2 or 3 CTAs per SM measured the same (config 3)
#endif
__global__ void __launch_bounds__(kSortThreads, SFG_BLKSORT_MINB) k_blk_sort(const uint32_t* __restrict__ tkey,
                                                      const float* __restrict__ tval,
                                                      const int32_t* __restrict__ off, int p, int64_t n,
                                                      int64_t nnz, int32_t* __restrict__ ptr,
                                                      int32_t* __restrict__ orow, float* __restrict__ oval) {
  constexpr int kPer = kBlkCap / kSortThreads;
  __shared__ int32_t cnt[kBlkCols + 1];
  __shared__ uint32_t scan_smem[34];
  __shared__ int32_t srow[kBlkCap];
  __shared__ float sval[kBlkCap];
  const int b = blockIdx.x;
  const int32_t s = off[(int64_t)b * p], size = off[(int64_t)(b + 1) * p] - s;
  const int64_t c0 = (int64_t)b << kBlkColBits;
  const int ncols = n - c0 < kBlkCols ? (int)(n - c0) : kBlkCols;
  for (int i = threadIdx.x; i < kBlkCols; i += kSortThreads) cnt[i] = 0;
  __syncthreads();
  int r[kPer], c[kPer], slot[kPer];
  float v[kPer];
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int i = k * kSortThreads + threadIdx.x;
    if (i < size) {
      const uint32_t key = tkey[s + i];
      r[k] = (int)(key >> kBlkColBits);
      c[k] = (int)(key & (kBlkCols - 1));
      v[k] = tval[s + i];
    }
  }
#pragma unroll
  for (int k = 0; k < kPer; ++k)
    if (k * kSortThreads + threadIdx.x < size) slot[k] = atomicAdd(&cnt[c[k]], 1);
  __syncthreads();
  // exclusive scan of the per-column counts (kBlkCols / kBlock per thread)
  constexpr int kColsPer = kBlkCols / kSortThreads;
  int loc[kColsPer], sum = 0;
#pragma unroll
  for (int q = 0; q < kColsPer; ++q) {
    loc[q] = cnt[threadIdx.x * kColsPer + q];
    sum += loc[q];
  }
  uint32_t tot;
  int run = (int)block_exclusive_scan<uint32_t, kSortThreads>((uint32_t)sum, scan_smem, &tot);
  int len[kColsPer];
#pragma unroll
  for (int q = 0; q < kColsPer; ++q) {
    len[q] = loc[q];
    cnt[threadIdx.x * kColsPer + q] = run;  // column start within the block
    run += loc[q];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kPer; ++k)
    if (k * kSortThreads + threadIdx.x < size) {
      const int pos = cnt[c[k]] + slot[k];
      srow[pos] = r[k];
      sval[pos] = v[k];
    }
  __syncthreads();
  // each column's rows in ascending order (columns are short; the reference
  // order is the stable sort of a row-sorted input)
#pragma unroll
  for (int q = 0; q < kColsPer; ++q) {
    const int st = cnt[threadIdx.x * kColsPer + q], n_ = len[q];
    for (int i = st + 1; i < st + n_; ++i) {
      const int rr = srow[i];
      const float vv = sval[i];
      int j = i - 1;
      while (j >= st && srow[j] > rr) {
        srow[j + 1] = srow[j];
        sval[j + 1] = sval[j];
        --j;
      }
      srow[j + 1] = rr;
      sval[j + 1] = vv;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < size; i += kSortThreads) {
    orow[s + i] = srow[i];
    oval[s + i] = sval[i];
  }
  for (int i = threadIdx.x; i < ncols; i += kSortThreads) ptr[c0 + i] = s + cnt[i];
  if (c0 + ncols == n && threadIdx.x == 0) ptr[n] = (int32_t)nnz;
}

int bits_for(int64_t extent) {
  int b = 0;
  while ((int64_t(1) << b) < extent) ++b;
  return b;
}

}  // namespace

// Column-block partition path (above); false when a block would exceed the
// shared-memory sort (then the caller takes the histogram path).
bool csc_by_column_blocks(sfg_context* ctx, const sfg_tensor* s, sfg_tensor* t) {
  const int64_t n = s->n, nnz = s->nnz;
  const int64_t nb = ceil_div(n, (int64_t)kBlkCols);
  if (nb > kMaxBlks || nb * kBlkCap < nnz) return false;  // some block would overflow anyway
  if (s->m > (int64_t(1) << (32 - kBlkColBits))) return false;  // rows travel in 22 bits
  const int p = kPartCtas;
  const int64_t cells = nb * p;
  int32_t* counts = dalloc_n<int32_t>(ctx, cells);
  int32_t* off = dalloc_n<int32_t>(ctx, cells + 1);
  int32_t* dummy = dalloc_n<int32_t>(ctx, cells);
  const int tiles = (int)ceil_div(cells, kTile);
  auto* status = lookback_status(ctx, tiles);
  auto* mx = static_cast<int32_t*>(scratch(ctx, 64));
  SFG_CUDA(cudaMemsetAsync(mx, 0, 8, ctx->stream));
  SFG_LAUNCH(k_blk_count, p, kBlock, 0, ctx->stream, s->idx, nnz, (int)nb, counts);
  SFG_LAUNCH(k_count_scan, tiles, kBlock, 0, ctx->stream, counts, (int32_t)cells, off, dummy, status,
             ctx->epoch++, mx + 1);
  SFG_LAUNCH(k_blk_max, (int)std::min<int64_t>(ceil_div(nb, kBlock), 64), kBlock, 0, ctx->stream, off, (int)nb, p,
             mx);
  // The scatter needs only the offsets: it is enqueued before the host
  // waits for the largest block size, so that round trip overlaps it (an
  // oversized block — rare — discards the scatter and takes the other path).
  read_back_start(ctx, mx, sizeof(int32_t));
  uint32_t* tkey = dalloc_n<uint32_t>(ctx, nnz);
  float* tval = dalloc_n<float>(ctx, nnz);
  SFG_LAUNCH(k_blk_scatter, p, kBlock, 0, ctx->stream, s->row, s->idx, static_cast<const float*>(s->val), nnz,
             (int)nb, off, tkey, tval);
  int32_t big = 0;
  read_back_wait(ctx, sizeof big, &big);
  if (big > kBlkCap) {
    for (void* q : {(void*)counts, (void*)off, (void*)dummy, (void*)tkey, (void*)tval}) dfree(ctx, q);
    return false;
  }
  SFG_LAUNCH(k_blk_sort, (int)nb, kSortThreads, 0, ctx->stream, tkey, tval, off, p, n, nnz, t->ptr, t->idx,
             static_cast<float*>(t->val));
  for (void* q : {(void*)counts, (void*)off, (void*)dummy, (void*)tkey, (void*)tval}) dfree(ctx, q);
  return true;
}

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
  if (csc_by_column_blocks(ctx, s, t)) return t;
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
