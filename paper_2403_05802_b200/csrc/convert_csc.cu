// convert_csc.cu — COO -> CSC.
//
// Reference: plan Swap(0,1) Sort Fill(0) Merge(0) (
// operators.hpp:234-241 Swap, 298-301 Sort = stable sort_entries,
// tensor.hpp:98-114). The result is uniquely determined: column pointers
// ptr[n+1], and within each column the rows in ascending order (the input
// is row-sorted and the sort is stable), materialized like CSR with the
// roles of rows and columns exchanged (storage.hpp:171-200).
//
// Device plan. (1) Column-bucket partition (every bucket of <= 8,192
// columns holds <= 22,528 entries, e.g. the hypersparse config 3): count
// per bucket, scan, scatter into bucket regions, sort each bucket in shared
// memory — below. (2) Otherwise, when every column holds <= kShortCol entries:
// column histogram (RED atomics) -> single-pass look-back scan ->
// atomic-cursor scatter -> per-column insertion sort by row, which restores
// the stable order. (3) Any longer column: stable LSD radix sort on the
// column bits with the row carried in the upper key half, then compression
// of the sorted columns. Config 3 (8.4 M entries, 4 M columns): (1) 0.21 ms,
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

// --------------------------------------------- column-bucket partition path
// Two passes, atomic-free in global memory and coalesced both ways.
// (0) Each of P CTAs counts its contiguous share of the entries per column
//     bucket (w consecutive columns) in shared memory; an exclusive scan over
//     (bucket, CTA) gives every CTA its write range inside every bucket.
// (1) Each CTA reorders its share, a tile of entries at a time, by bucket
//     in shared memory and writes each bucket's run to the bucket's range:
//     consecutive threads write consecutive addresses. The intermediate
//     (row, value, column-in-bucket: 10 B an entry) is kept in L2 for pass 2.
// (2) One CTA per bucket loads its <= kSortPer x threads entries, counts
//     them per column, places them by column, insertion-sorts each (short) column by
//     row — the stable order of the row-sorted input — and writes idx / val
//     / ptr of its columns with coalesced stores.
constexpr int kPartThreads = 512;
constexpr int kPartPer = 24;        // pass-1 entries per thread per round (32 when shared memory allows)
constexpr int kMaxBuckets = 4096;
constexpr int kMaxBucketCols = 8192;  // columns per bucket
constexpr int kSortPer = 22;        // pass-2 entries per thread

// Bucket of column c < 2^31: c / w as a multiply-high, m = ceil(2^k / w) with
// k = 31 + ceil(log2 w) (then m < 2^32 and c * (m * w - 2^k) < 2^k, so the
// quotient is exact).
struct BucketDiv {
  uint32_t w, m;
  int k;
  __device__ __forceinline__ uint32_t operator()(int32_t c) const {
    return (uint32_t)(((uint64_t)(uint32_t)c * m) >> k);
  }
};
BucketDiv bucket_div(uint32_t w) {
  int l = 0;
  while ((uint64_t(1) << l) < w) ++l;
  const int k = 31 + l;
  return {w, (uint32_t)(((uint64_t(1) << k) + w - 1) / w), k};
}

// Entries [e0, e1) of pass-1 CTA `cta`: equal shares rounded up to a
// multiple of 4, so each share starts 16-byte aligned (k_bkt_count and
// k_bkt_part must agree on them: the bucket offsets are per CTA).
__device__ __forceinline__ void part_range(int64_t nnz, int cta, int ctas, int64_t& e0, int64_t& e1) {
  const int64_t per = ((nnz + ctas - 1) / ctas + 3) & ~int64_t(3);
  e0 = min(nnz, cta * per);
  e1 = min(nnz, e0 + per);
}

// kVec: the input arrays are 16-byte aligned (int4 loads, four entries each)
template <bool kVec>
__global__ void __launch_bounds__(kPartThreads) k_bkt_count(const int32_t* __restrict__ col, int64_t nnz, BucketDiv bkt,
                                                             int nb, int32_t* __restrict__ counts,
                                                             int32_t* __restrict__ btot, uint32_t* __restrict__ done,
                                                             int32_t* __restrict__ mx) {
  __shared__ int32_t h[kMaxBuckets];
  __shared__ bool last;
  for (int i = threadIdx.x; i < nb; i += kPartThreads) h[i] = 0;
  __syncthreads();
  int64_t e0, e1;
  part_range(nnz, blockIdx.x, gridDim.x, e0, e1);
  constexpr int U = 8;  // loads in flight per thread
  int64_t e = e0 + threadIdx.x;
  if constexpr (kVec) {
    const int64_t nv = (e1 - e0) >> 2;
    const int4* c4 = reinterpret_cast<const int4*>(col + e0);
    // double-buffered: the next batch's loads are in flight while this
    // batch is counted
    int4 q[U], nq[U];
    auto load = [&](int4 (&dst)[U], int64_t j) {
#pragma unroll
      for (int u = 0; u < U; ++u)
        dst[u] = j + u * kPartThreads < nv ? ld_stream(c4 + j + u * kPartThreads) : make_int4(-1, -1, -1, -1);
    };
    load(q, threadIdx.x);
    for (int64_t j = threadIdx.x; j < nv; j += U * kPartThreads) {
      if (j + U * kPartThreads < nv) load(nq, j + U * kPartThreads);
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (q[u].x >= 0) {
          atomicAdd(&h[bkt(q[u].x)], 1);
          atomicAdd(&h[bkt(q[u].y)], 1);
          atomicAdd(&h[bkt(q[u].z)], 1);
          atomicAdd(&h[bkt(q[u].w)], 1);
        }
#pragma unroll
      for (int u = 0; u < U; ++u) q[u] = nq[u];
    }
    e = e0 + nv * 4 + threadIdx.x;
  }
  for (; e < e1; e += U * kPartThreads) {
    int c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = e + u * kPartThreads < e1 ? ld_stream(col + e + u * kPartThreads) : -1;
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (c[u] >= 0) atomicAdd(&h[bkt(c[u])], 1);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nb; b += kPartThreads) {
    counts[(int64_t)b * gridDim.x + blockIdx.x] = h[b];
    if (h[b]) atomicAdd(btot + b, h[b]);
  }
  // the last CTA to finish takes the largest bucket (btot, done and mx are
  // zeroed by the caller) for the host's pass-2 capacity check
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (last) {
    __threadfence();
    int m = 0;
    for (int b = threadIdx.x; b < nb; b += kPartThreads) m = max(m, __ldcg(btot + b));
    m = warp_max(m);
    if ((threadIdx.x & 31) == 0) atomicMax(mx, m);
  }
}

// Pass 1. Dynamic shared memory: row, value, column of kPartTile entries,
// then per-bucket count, start and write cursor.
// kPer entries per thread per round (the tile: as large as the shared memory
// left by the bucket counters allows)
template <bool kVec, int kPer>
__global__ void __launch_bounds__(kPartThreads, 1) k_bkt_part(const int32_t* __restrict__ row,
                                                               const int32_t* __restrict__ col,
                                                               const float* __restrict__ val, int64_t nnz,
                                                               BucketDiv bkt, int nb, const int32_t* __restrict__ off,
                                                               int32_t* __restrict__ trow, float* __restrict__ tval,
                                                               uint16_t* __restrict__ tcol) {
  constexpr int kPartTile = kPartThreads * kPer;
  extern __shared__ int32_t sm[];
  int32_t* s_row = sm;
  float* s_val = reinterpret_cast<float*>(sm + kPartTile);
  int32_t* s_col = sm + 2 * kPartTile;
  int32_t* s_cnt = sm + 3 * kPartTile;
  int32_t* s_start = s_cnt + nb;
  int32_t* s_cur = s_start + nb;
  __shared__ uint32_t scan_smem[34];
  const int tid = threadIdx.x;
  for (int b = tid; b < nb; b += kPartThreads) s_cur[b] = off[(int64_t)b * gridDim.x + blockIdx.x];
  const uint64_t once = l2_evict_first(), keep = l2_evict_last();
  int64_t e0, e1;
  part_range(nnz, blockIdx.x, gridDim.x, e0, e1);
  constexpr int kBPer = kMaxBuckets / kPartThreads;  // buckets per thread in the scan
  // slot k of this thread is tile entry item(k); with kVec, four
  // consecutive entries per int4 load (order within a bucket run does not
  // matter: pass 2 sorts each column by row). Only the columns are held in
  // registers — the next tile's are loaded while this tile's runs are
  // written out; rows and values are loaded after the scan, straight into
  // their places.
  auto item = [&](int k) { return kVec ? 4 * ((k >> 2) * kPartThreads + tid) + (k & 3) : k * kPartThreads + tid; };
  int c[kPer], rank[kPer];
  auto load_cols = [&](int64_t base, int cnt) {
    if constexpr (kVec) {
#pragma unroll
      for (int g = 0; g < kPer / 4; ++g) {
        const int i = 4 * (g * kPartThreads + tid);
        if (i + 3 < cnt) {
          const int4 cq = ld_stream(reinterpret_cast<const int4*>(col + base + i));
          c[4 * g] = cq.x, c[4 * g + 1] = cq.y, c[4 * g + 2] = cq.z, c[4 * g + 3] = cq.w;
        } else {
#pragma unroll
          for (int t = 0; t < 4; ++t)
            if (i + t < cnt) c[4 * g + t] = ld_stream(col + base + i + t);
        }
      }
    } else {
#pragma unroll
      for (int k = 0; k < kPer; ++k)
        if (item(k) < cnt) c[k] = (int)ld_hint(col + base + item(k), once);
    }
  };
  auto tile_len = [&](int64_t base) { return (int)(e1 - base < kPartTile ? e1 - base : kPartTile); };
  if (e0 < e1) load_cols(e0, tile_len(e0));
  for (int64_t base = e0; base < e1; base += kPartTile) {
    const int cnt = tile_len(base);
    for (int b = tid; b < nb; b += kPartThreads) s_cnt[b] = 0;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kPer; ++k)
      if (item(k) < cnt) rank[k] = atomicAdd(&s_cnt[bkt(c[k])], 1);
    __syncthreads();
    int loc[kBPer], sum = 0;
#pragma unroll
    for (int q = 0; q < kBPer; ++q) {
      const int b = tid * kBPer + q;
      loc[q] = b < nb ? s_cnt[b] : 0;
      sum += loc[q];
    }
    uint32_t tot;
    int run = (int)block_exclusive_scan<uint32_t, kPartThreads>((uint32_t)sum, scan_smem, &tot);
#pragma unroll
    for (int q = 0; q < kBPer; ++q) {
      const int b = tid * kBPer + q;
      if (b < nb) s_start[b] = run;
      run += loc[q];
    }
    __syncthreads();
    if constexpr (kVec) {
#pragma unroll
      for (int g = 0; g < kPer / 4; ++g) {
        const int i = 4 * (g * kPartThreads + tid);
        int r[4];
        float v[4];
        if (i + 3 < cnt) {
          const int4 rq = ld_stream(reinterpret_cast<const int4*>(row + base + i));
          const float4 vq = ld_stream(reinterpret_cast<const float4*>(val + base + i));
          r[0] = rq.x, r[1] = rq.y, r[2] = rq.z, r[3] = rq.w;
          v[0] = vq.x, v[1] = vq.y, v[2] = vq.z, v[3] = vq.w;
        } else {
#pragma unroll
          for (int t = 0; t < 4; ++t)
            if (i + t < cnt) r[t] = ld_stream(row + base + i + t), v[t] = ld_stream(val + base + i + t);
        }
#pragma unroll
        for (int t = 0; t < 4; ++t)
          if (i + t < cnt) {
            const int k = 4 * g + t, pos = s_start[bkt(c[k])] + rank[k];
            s_row[pos] = r[t];
            s_val[pos] = v[t];
            s_col[pos] = c[k];
          }
      }
    } else {
#pragma unroll
      for (int k = 0; k < kPer; ++k)
        if (item(k) < cnt) {
          const int pos = s_start[bkt(c[k])] + rank[k];
          s_row[pos] = (int)ld_hint(row + base + item(k), once);
          s_val[pos] = __uint_as_float(ld_hint(val + base + item(k), once));
          s_col[pos] = c[k];
        }
    }
    __syncthreads();
    if (base + kPartTile < e1) load_cols(base + kPartTile, tile_len(base + kPartTile));
    // bucket runs out: consecutive positions of a bucket go to consecutive
    // addresses of the bucket's range
    for (int p = tid; p < cnt; p += kPartThreads) {
      const int cc = s_col[p], b = bkt(cc);
      const int64_t dst = (int64_t)s_cur[b] + (p - s_start[b]);
      st_hint(trow + dst, (uint32_t)s_row[p], keep);
      st_hint(tval + dst, __float_as_uint(s_val[p]), keep);
      tcol[dst] = (uint16_t)(cc - b * (int)bkt.w);
    }
    __syncthreads();
    for (int b = tid; b < nb; b += kPartThreads) s_cur[b] += s_cnt[b];
  }
}

// Pass 2: a CTA per bucket. Static shared memory: sorted rows and values of
// <= kBucketCap entries, per-column counts / starts.
template <int kSortThreads, int kMinBlocks>
__global__ void __launch_bounds__(kSortThreads, kMinBlocks) k_bkt_sort(const int32_t* __restrict__ trow,
                                                               const float* __restrict__ tval,
                                                               const uint16_t* __restrict__ tcol,
                                                               const int32_t* __restrict__ off, int p, int w,
                                                               int64_t n, int64_t nnz, int32_t* __restrict__ ptr,
                                                               int32_t* __restrict__ orow, float* __restrict__ oval) {
  constexpr int kBucketCap = kSortThreads * kSortPer;
  extern __shared__ int32_t sm2[];  // cnt[w] | srow[kBucketCap] | sval[kBucketCap]
  int32_t* cnt = sm2;
  int32_t* srow = sm2 + w;
  float* sval = reinterpret_cast<float*>(srow + kBucketCap);
  __shared__ uint32_t scan_smem[34];
  const int b = blockIdx.x;
  const int ncols_b = w;
  const int32_t s = off[(int64_t)b * p], size = off[(int64_t)(b + 1) * p] - s;
  const int64_t c0 = (int64_t)b * w;
  const int ncols = n - c0 < ncols_b ? (int)(n - c0) : ncols_b;
  for (int i = threadIdx.x; i < ncols_b; i += kSortThreads) cnt[i] = 0;
  __syncthreads();
  // per entry: (slot within its column << 16 | column); rows and values are
  // loaded once the column starts are known, straight into their places
  int cs[kSortPer];
#pragma unroll
  for (int k = 0; k < kSortPer; ++k) {
    const int i = k * kSortThreads + threadIdx.x;
    if (i < size) cs[k] = tcol[s + i];
  }
#pragma unroll
  for (int k = 0; k < kSortPer; ++k)
    if (k * kSortThreads + threadIdx.x < size) cs[k] |= atomicAdd(&cnt[cs[k]], 1) << 16;
  __syncthreads();
  // exclusive scan of the per-column counts; each thread owns a run of
  // columns (ceil(ncols_b / kSortThreads))
  const int per = (ncols_b + kSortThreads - 1) / kSortThreads;
  const int cbeg = threadIdx.x * per;
  int sum = 0;
  for (int q = 0; q < per; ++q) sum += cbeg + q < ncols_b ? cnt[cbeg + q] : 0;
  uint32_t tot;
  int run = (int)block_exclusive_scan<uint32_t, kSortThreads>((uint32_t)sum, scan_smem, &tot);
  __syncthreads();
  for (int q = 0; q < per; ++q)
    if (cbeg + q < ncols_b) {
      const int l = cnt[cbeg + q];
      cnt[cbeg + q] = run;  // column start within the bucket
      run += l;
    }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kSortPer; ++k) {
    const int i = k * kSortThreads + threadIdx.x;
    if (i < size) {
      const int pos = cnt[cs[k] & 0xffff] + (cs[k] >> 16);
      srow[pos] = trow[s + i];
      sval[pos] = tval[s + i];
    }
  }
  __syncthreads();
  // each column's rows in ascending order (columns are short; the reference
  // order is the stable sort of a row-sorted input)
  for (int q = 0; q < per; ++q) {
    const int cq = cbeg + q;
    if (cq >= ncols_b) break;
    const int st = cnt[cq], en = cq + 1 < ncols_b ? cnt[cq + 1] : size;
    for (int i = st + 1; i < en; ++i) {
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

// Column-bucket partition path (above); false when no bucket width fits
// the shared-memory sort (then the caller takes the histogram path).
bool csc_by_column_buckets(sfg_context* ctx, const sfg_tensor* s, sfg_tensor* t) {
  const int64_t n = s->n, nnz = s->nnz;
  // fewest buckets (longest pass-1 runs) whose average fill is at most 3/4
  // of a pass-2 CTA's capacity, with <= max_cols columns per bucket; a
  // count of several waves is rounded up to whole pass-2 waves.
  // Pass 2: one 1,024-thread CTA per SM (22,528 entries per bucket), or with
  // SFG_CSC_SORT=512 two 512-thread CTAs per SM (11,264 entries)
  const char* sort_env = getenv("SFG_CSC_SORT");
  const int sort_threads = sort_env && atoi(sort_env) == 512 ? 512 : 1024;
  const int64_t cap = (int64_t)sort_threads * kSortPer, max_cols = sort_threads == 512 ? 4096 : kMaxBucketCols;
  const int64_t kAvgFill = cap * 3 / 4;
  const int p = ctx->sms;  // one pass-1 CTA per SM
  const int wave = sort_threads == 512 ? 2 * p : p;
  int64_t nb = std::max(ceil_div(nnz, kAvgFill), ceil_div(n, max_cols));
  if (nb > wave / 2) nb = ceil_div(nb, int64_t(wave)) * wave;
  const int64_t w = ceil_div(n, nb);
  nb = ceil_div(n, w);
  const BucketDiv bkt = bucket_div((uint32_t)w);
  if (nb > kMaxBuckets || nb * kAvgFill < nnz) return false;
  const int64_t cells = nb * p;
  int32_t* counts = dalloc_n<int32_t>(ctx, cells);
  int32_t* off = dalloc_n<int32_t>(ctx, cells + 1);
  int32_t* dummy = dalloc_n<int32_t>(ctx, cells);
  const int tiles = (int)ceil_div(cells, kTile);
  auto* status = lookback_status(ctx, tiles);
  // scratch: [0] largest bucket, [1] largest cell (the scan's), [2] CTAs
  // done counting, [16, 16 + nb) bucket totals
  auto* mx = static_cast<int32_t*>(scratch(ctx, 64 + 4 * nb));
  SFG_CUDA(cudaMemsetAsync(mx, 0, 64 + 4 * nb, ctx->stream));
  int32_t* btot = mx + 16;
  auto* done = reinterpret_cast<uint32_t*>(mx + 2);
  const bool vec = ((reinterpret_cast<uintptr_t>(s->row) | reinterpret_cast<uintptr_t>(s->idx) |
                     reinterpret_cast<uintptr_t>(s->val)) & 15) == 0;
  if (vec)
    SFG_LAUNCH(k_bkt_count<true>, p, kPartThreads, 0, ctx->stream, s->idx, nnz, bkt, (int)nb, counts, btot, done,
               mx);
  else
    SFG_LAUNCH(k_bkt_count<false>, p, kPartThreads, 0, ctx->stream, s->idx, nnz, bkt, (int)nb, counts, btot, done,
               mx);
  // the largest bucket is known after the count: its read-back starts now,
  // and the scan and pass 1 (which needs only the offsets) are enqueued
  // before the host waits for it, so that round trip overlaps them (an
  // oversized bucket — rare — discards pass 1 and takes the other path)
  read_back_start(ctx, mx, sizeof(int32_t));
  SFG_LAUNCH(k_count_scan, tiles, kBlock, 0, ctx->stream, counts, (int32_t)cells, off, dummy, status,
             ctx->epoch++, mx + 1);
  int32_t* trow = dalloc_n<int32_t>(ctx, nnz);
  float* tval = dalloc_n<float>(ctx, nnz);
  uint16_t* tcol = dalloc_n<uint16_t>(ctx, nnz);
  // pass-1 tile: 16,384 entries when the bucket counters leave room, else 12,288
  const bool big_tile = (size_t)3 * kPartThreads * 32 * 4 + (size_t)3 * nb * 4 <= 227 * 1024;
  const size_t smem = (size_t)3 * kPartThreads * (big_tile ? 32 : kPartPer) * 4 + (size_t)3 * nb * 4;
  const float* sv = static_cast<const float*>(s->val);
#define SFG_BKT_PART(V, P)                                                                                    \
  do {                                                                                                        \
    const auto k_bkt_part_ = k_bkt_part<V, P>;                                                                \
    SFG_CUDA(cudaFuncSetAttribute(k_bkt_part_, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));      \
    SFG_LAUNCH(k_bkt_part_, p, kPartThreads, smem, ctx->stream, s->row, s->idx, sv, nnz, bkt, (int)nb, off,              \
               trow, tval, tcol);                                                                             \
  } while (0)
  if (vec && big_tile) SFG_BKT_PART(true, 32);
  else if (vec) SFG_BKT_PART(true, kPartPer);
  else if (big_tile) SFG_BKT_PART(false, 32);
  else SFG_BKT_PART(false, kPartPer);
#undef SFG_BKT_PART
  int32_t big = 0;
  read_back_wait(ctx, sizeof big, &big);
  auto release = [&] {
    for (void* q : {(void*)counts, (void*)off, (void*)dummy, (void*)trow, (void*)tval, (void*)tcol}) dfree(ctx, q);
  };
  if (big > cap) {
    release();
    return false;
  }
  const size_t smem2 = ((size_t)w + 2 * cap) * 4;
  if (sort_threads == 512) {
    const auto k_bkt_sort_ = k_bkt_sort<512, 2>;
    SFG_CUDA(cudaFuncSetAttribute(k_bkt_sort_, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
    SFG_LAUNCH(k_bkt_sort_, (int)nb, 512, smem2, ctx->stream, trow, tval, tcol, off, p, (int)w, n, nnz,
               t->ptr, t->idx, static_cast<float*>(t->val));
  } else {
    const auto k_bkt_sort_ = k_bkt_sort<1024, 1>;
    SFG_CUDA(cudaFuncSetAttribute(k_bkt_sort_, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
    SFG_LAUNCH(k_bkt_sort_, (int)nb, 1024, smem2, ctx->stream, trow, tval, tcol, off, p, (int)w, n, nnz,
               t->ptr, t->idx, static_cast<float*>(t->val));
  }
  release();
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
  if (csc_by_column_buckets(ctx, s, t)) return t;
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

// DCSC: map (d1, d0); merge(0), trim(0,1) (formats.hpp:43), plan Swap(0,1)
// Sort Merge(0): the CSC with its empty columns dropped — L0 idx = the
// nonempty columns ascending (bounds [0, n-1]), L1 ptr over them + the rows.
// Device: the CSC conversion above, then a flag / scan / scatter over the
// column pointers (the row and value arrays are taken over as they are).
namespace {

__global__ void k_col_nonempty(const int32_t* __restrict__ ptr, int64_t n, int32_t* __restrict__ flag) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x)
    flag[c] = __ldg(ptr + c + 1) > __ldg(ptr + c) ? 1 : 0;
}

__global__ void k_col_compact(const int32_t* __restrict__ ptr, const int32_t* __restrict__ base, int64_t n,
                              int32_t* __restrict__ cols, int32_t* __restrict__ dptr) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x) {
    const int32_t b = __ldg(base + c);
    if (__ldg(base + c + 1) > b) {
      cols[b] = (int32_t)c;
      dptr[b] = __ldg(ptr + c);
    }
    if (c == n - 1) dptr[__ldg(base + n)] = __ldg(ptr + n);
  }
}

}  // namespace

sfg_tensor* coo_to_dcsc(sfg_context* ctx, const sfg_tensor* s) {
  sfg_tensor* csc = coo_to_csc(ctx, s);
  const int64_t n = s->n;
  sfg_tensor* t = new_tensor(ctx, SFG_DCSC, s->m, n);
  t->nnz = csc->nnz;
  t->idx = csc->idx;
  t->val = csc->val;
  csc->idx = nullptr;
  csc->val = nullptr;
  int32_t* flag = dalloc_n<int32_t>(ctx, n);
  int32_t* base = dalloc_n<int32_t>(ctx, n + 1);
  SFG_LAUNCH(k_col_nonempty, stream_grid(ctx, n, kBlock, 4, 8), kBlock, 0, ctx->stream, csc->ptr, n, flag);
  scan_counts(ctx, flag, n, base);
  int32_t nnc = 0;
  read_back(ctx, base + n, sizeof nnc, &nnc);
  t->row = dalloc_n<int32_t>(ctx, nnc);
  t->ptr = dalloc_n<int32_t>(ctx, nnc + 1);
  t->nnr = nnc;
  SFG_LAUNCH(k_col_compact, stream_grid(ctx, n, kBlock, 4, 8), kBlock, 0, ctx->stream, csc->ptr, base, n, t->row,
             t->ptr);
  dfree(ctx, flag);
  dfree(ctx, base);
  free_tensor_arrays(csc);
  delete csc;
  return t;
}

}  // namespace sfg
