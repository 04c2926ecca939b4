// convert_bcsr.cu — COO -> BCSR(r, c).
//
// Reference: plan TileSplit(0,r) TileSplit(2,c) Swap(1,2) Sort Fill(3)
// Fill(2) Fill(0) Vectorize(2) Merge(0). TileSplit
// (operators.hpp:263-285) maps (d0, d1) -> (d0/r, d1/c, d0%r, d1%c); the
// mod level's bounds are [0, r-1] unless the whole range lies in one tile,
// in which case they are [lo%r, hi%r] — a single block row is only M rows
// tall (likewise for columns). Fill(3), Fill(2) complete every touched
// block with zeros, positions past M/N included (operators.hpp:346-379);
// Fill(0) leaves empty block rows as empty ptr runs. Materialized: L0 size
// (block rows), L1 ptr[nbr+1] + idx[nblocks] (block columns, ascending),
// L2/L3 dense, values block-major and row-major inside a block
// (storage.hpp:142-218).
//
// Device plan: (1) block-row pointers from the sorted rows; (2) one CTA per
// block row marks its block columns in a shared-memory bitmap (restricted
// to the row's [min, max] block-column range) and counts them; (3)
// look-back scan of the counts -> L1.ptr; (4) zero-fill the value array;
// (5) each CTA rebuilds its bitmap, ranks the set bits (block index =
// prefix popcount), writes L1.idx and scatters every entry into its block.
#include <cuda_bf16.h>

#include "devutil.cuh"
#include "internal.cuh"

namespace sfg {

namespace {

constexpr int kBlock = 256;
constexpr int kMaxWords = 24 * 1024;  // 96 KB bitmap (+96 KB prefix) => <= 786K block columns

// x / d for x >= 0, a shift when d is a power of two (the block sizes in
// practice; a division by a run-time divisor costs ~20 instructions)
__device__ __forceinline__ int pow2_shift(int d) { return (d & (d - 1)) == 0 ? __ffs(d) - 1 : -1; }
__device__ __forceinline__ int divp(int x, int d, int sh) { return sh >= 0 ? x >> sh : x / d; }

// Block-row pointers: the row pointers of the block-row ids (row / r) of
// the sorted entries — the CSR row-pointer pass (devutil.cuh: 16-byte row
// loads, warp-staged lower-bound searches, coalesced stores).
constexpr int kBrowVec = 4;

__global__ void __launch_bounds__(kBlock) k_brow_ptr(const int32_t* __restrict__ row, int64_t nnz,
                                                      int32_t r, int32_t nbr,
                                                      int32_t* __restrict__ bptr) {
  constexpr int kChunk = 128 * kBrowVec;
  __shared__ __align__(16) int32_t s_rows[kBlock / 32][kChunk];
  const int rs = pow2_shift(r);
  const int64_t nchunk = (nnz + kChunk - 1) / kChunk;
  const int64_t warps = (int64_t)gridDim.x * (kBlock / 32);
  for (int64_t ch = (int64_t)blockIdx.x * (kBlock / 32) + (threadIdx.x >> 5); ch < nchunk; ch += warps) {
    const int64_t base = ch * kChunk;
    RowChunk<kBrowVec> c;
    load_row_chunk(row, nnz, base, c);
#pragma unroll
    for (int g = 0; g < kBrowVec; ++g)
#pragma unroll
      for (int i = 0; i < 4; ++i) c.r[g][i] = divp(c.r[g][i], r, rs);
    c.prev = c.prev < 0 ? -1 : divp(c.prev, r, rs);
    chunk_row_ptr(c, nnz, base, nbr, s_rows[threadIdx.x >> 5], bptr);
  }
}

// Bitmap of the block columns present in block row `br` over [lo, hi].
// Four entries per thread per step, loads first (the loop is latency
// bound). (Skipping entries whose block column repeats its predecessor's,
// or an OR-scan per run of equal words with one atomic per run, both
// measured slower in round 1: 391 / 451 vs 290 us for the count kernel at
// 32768^2; the match-any aggregation below is faster for wide blocks.)
__device__ __forceinline__ void mark(const int32_t* __restrict__ col, int32_t s, int32_t e,
                                     int32_t c, int32_t lo, uint32_t* bm) {
  constexpr int U = 4;
  const int cs = pow2_shift(c);
  // warp-uniform trip count: the warp-wide match / reduce below need every lane
  for (int32_t kw = s + (int32_t)(threadIdx.x & ~31u); kw < e; kw += U * blockDim.x) {
    const int32_t k = kw + (int32_t)(threadIdx.x & 31);
    int v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = k + u * (int32_t)blockDim.x < e ? __ldg(col + k + u * blockDim.x) : -1;
    if (c >= 8) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        // lanes marking the same word OR their bits first: one shared atomic
        // per distinct word of the warp (a row's consecutive entries share
        // their block column). 16 x 16 at 32768^2: count 365 -> ~220 us;
        // with 4-wide blocks the match costs more than it saves.
        const int b = v[u] >= 0 ? divp(v[u], c, cs) - lo : -32 - (int)(threadIdx.x & 31);
        const int wd = b >> 5;
        const unsigned peers = __match_any_sync(kFull, wd);
        const uint32_t bits = __reduce_or_sync(peers, v[u] >= 0 ? 1u << (b & 31) : 0u);
        if (v[u] >= 0 && (int)(threadIdx.x & 31) == __ffs(peers) - 1) atomicOr(bm + wd, bits);
      }
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (v[u] >= 0) {
          const int b = divp(v[u], c, cs) - lo;
          atomicOr(bm + (b >> 5), 1u << (b & 31));
        }
    }
  }
}

__device__ __forceinline__ void col_range(const int32_t* __restrict__ col, int32_t s, int32_t e,
                                          int32_t c, int* smin, int* smax, int32_t* lo,
                                          int32_t* hi) {
  int mn = INT32_MAX, mx = -1;
  for (int32_t k = s + threadIdx.x; k < e; k += blockDim.x) {
    int b = divp(__ldg(col + k), c, pow2_shift(c));
    mn = min(mn, b);
    mx = max(mx, b);
  }
  for (int o = 16; o > 0; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(kFull, mn, o));
    mx = max(mx, __shfl_xor_sync(kFull, mx, o));
  }
  if (threadIdx.x == 0) {
    *smin = INT32_MAX;
    *smax = -1;
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) {
    atomicMin(smin, mn);
    atomicMax(smax, mx);
  }
  __syncthreads();
  *lo = *smin;
  *hi = *smax;
}

// A block-column grid this narrow is marked over its whole range: no
// separate min/max pass over the columns.
constexpr int32_t kFullRangeCols = 32768;

// Block-count rule of the hybrid decompose (convert_bell.cu): per block row,
// a shared counter per block column gathers the nonzero
// count of every r x c block — a warp's 32 consecutive entries split into
// runs of one block column (a row's columns ascend), one shared atomic per
// run — then every entry is flagged by its block's count. Entries stay in
// place, so the flags are in input order.
constexpr int32_t kDecCounters = 48 * 1024;  // 192 KB of counters

__global__ void __launch_bounds__(kBlock) k_block_nz_flags(const int32_t* __restrict__ bptr,
                                                           const int32_t* __restrict__ col,
                                                           const float* __restrict__ val, int32_t c, int32_t nbr,
                                                           int32_t nbc, int64_t min_sum, bool count_values,
                                                           uint8_t* __restrict__ flag) {
  extern __shared__ uint32_t cnt[];  // nbc <= kDecCounters (host)
  const int lane = threadIdx.x & 31;
  const int cs = pow2_shift(c);
  for (int32_t br = blockIdx.x; br < nbr; br += gridDim.x) {
    const int32_t s = __ldg(bptr + br), e = __ldg(bptr + br + 1);
    if (s == e) continue;
    for (int w = threadIdx.x; w < nbc; w += blockDim.x) cnt[w] = 0;
    __syncthreads();
    for (int32_t k0 = s; k0 < e; k0 += blockDim.x) {
      const int32_t k = k0 + threadIdx.x;
      const bool in = k < e;
      const int b = in ? divp(__ldg(col + k), c, cs) : -1;
      const bool nz = in && (!count_values || __ldg(val + k) != 0.f);
      const int pb = __shfl_up_sync(kFull, b, 1);
      const bool head = in && (lane == 0 || pb != b);
      const unsigned hm = __ballot_sync(kFull, head), nm = __ballot_sync(kFull, nz);
      if (head) {
        const unsigned above = hm & ~((2u << lane) - 1u);
        const int h = above ? __ffs(above) - 1 : 32;
        const unsigned run = (h == 32 ? kFull : ((1u << h) - 1u)) & ~((1u << lane) - 1u);
        const int q = __popc(nm & run);
        if (q) atomicAdd(cnt + b, (uint32_t)q);
      }
    }
    __syncthreads();
    for (int32_t k = s + threadIdx.x; k < e; k += blockDim.x)
      flag[k] = (int64_t)cnt[divp(__ldg(col + k), c, cs)] >= min_sum ? 1 : 0;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kBlock) k_count_blocks(const int32_t* __restrict__ bptr,
                                                          const int32_t* __restrict__ col,
                                                          int32_t c, int32_t nbr, int32_t nbc,
                                                          uint32_t* __restrict__ gbm,
                                                          int32_t* __restrict__ cnt) {
  extern __shared__ uint32_t bm[];
  __shared__ int smin, smax, ssum;
  for (int32_t br = blockIdx.x; br < nbr; br += gridDim.x) {
    int32_t s = __ldg(bptr + br), e = __ldg(bptr + br + 1);
    if (s == e) {
      if (threadIdx.x == 0) cnt[br] = 0;
      continue;
    }
    int32_t lo = 0, hi = nbc - 1;
    if (nbc > kFullRangeCols) col_range(col, s, e, c, &smin, &smax, &lo, &hi);
    // words <= kMaxWords: the host rejects block grids wider than the bitmap
    // before launching (coo_to_bcsr), so there is no skip path here (which
    // would have to pass the same barriers as the marking path)
    int words = ((hi - lo) >> 5) + 1;
    for (int w = threadIdx.x; w < words; w += blockDim.x) bm[w] = 0;
    if (threadIdx.x == 0) ssum = 0;
    __syncthreads();
    mark(col, s, e, c, lo, bm);
    __syncthreads();
    int pc = 0;
    for (int w = threadIdx.x; w < words; w += blockDim.x) {
      pc += __popc(bm[w]);
      if (gbm) gbm[(int64_t)br * words + w] = bm[w];  // full-range bitmaps only: the fill reuses them
    }
    pc = warp_sum(pc);
    if ((threadIdx.x & 31) == 0) atomicAdd(&ssum, pc);
    __syncthreads();
    if (threadIdx.x == 0) cnt[br] = ssum;
    __syncthreads();
  }
}

constexpr int kItems = 16;
constexpr int kTile = kBlock * kItems;

__global__ void __launch_bounds__(kBlock) k_scan_i32(const int32_t* __restrict__ cnt, int32_t n,
                                                      int32_t* __restrict__ ptr,
                                                      unsigned long long* __restrict__ status,
                                                      uint32_t epoch) {
  __shared__ uint32_t smem[34];
  __shared__ uint32_t slot;
  const int64_t c0 = (int64_t)blockIdx.x * kTile + (int64_t)threadIdx.x * kItems;
  uint32_t v[kItems], sum = 0;
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    v[i] = c0 + i < n ? (uint32_t)__ldg(cnt + c0 + i) : 0u;
    sum += v[i];
  }
  uint32_t total;
  uint32_t excl = block_exclusive_scan<uint32_t, kBlock>(sum, smem, &total);
  uint32_t p = lookback_prefix(status, epoch, blockIdx.x, total, &slot) + excl;
#pragma unroll
  for (int i = 0; i < kItems; ++i)
    if (c0 + i < n) {
      ptr[c0 + i] = (int32_t)p;
      p += v[i];
    }
  if (c0 + kItems >= n && c0 < n) ptr[n] = (int32_t)p;
}

template <typename T>
__device__ __forceinline__ T to_val(float v);
template <>
__device__ __forceinline__ float to_val<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 to_val<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

template <typename T>
__global__ void __launch_bounds__(kBlock) k_fill_blocks(
    const int32_t* __restrict__ bptr, const int32_t* __restrict__ row,
    const int32_t* __restrict__ col, const float* __restrict__ val, int32_t r, int32_t c,
    int32_t rb, int32_t cb, int32_t nbr, int32_t nbc, const uint32_t* __restrict__ gbm,
    const int32_t* __restrict__ blk_ptr,
    int32_t* __restrict__ bidx, T* __restrict__ bval) {
  extern __shared__ uint32_t bm[];  // [words] bitmap, then [words] prefix
  __shared__ int smin, smax;
  __shared__ uint32_t wsum[34];
  const int cs = pow2_shift(c);
  for (int32_t br = blockIdx.x; br < nbr; br += gridDim.x) {
    int32_t s = __ldg(bptr + br), e = __ldg(bptr + br + 1);
    if (s == e) continue;
    int32_t lo = 0, hi = nbc - 1;
    if (nbc > kFullRangeCols) col_range(col, s, e, c, &smin, &smax, &lo, &hi);
    int words = ((hi - lo) >> 5) + 1;
    uint32_t* pre = bm + words;
    if (gbm) {  // the count kernel's bitmap of this block row
      for (int w = threadIdx.x; w < words; w += blockDim.x) bm[w] = gbm[(int64_t)br * words + w];
    } else {
      for (int w = threadIdx.x; w < words; w += blockDim.x) bm[w] = 0;
      __syncthreads();
      mark(col, s, e, c, lo, bm);
    }
    __syncthreads();
    // exclusive prefix of popcounts over the words: each thread owns a
    // contiguous run of words
    int per = (words + blockDim.x - 1) / blockDim.x;
    int w0 = threadIdx.x * per, w1 = min(words, w0 + per);
    uint32_t mine = 0;
    for (int w = w0; w < w1; ++w) mine += __popc(bm[w]);
    uint32_t tot;
    uint32_t ex = block_exclusive_scan<uint32_t, kBlock>(mine, wsum, &tot);
    for (int w = w0; w < w1; ++w) {
      pre[w] = ex;
      ex += __popc(bm[w]);
    }
    __syncthreads();
    const int32_t base = __ldg(blk_ptr + br);
    // L1.idx: block columns in ascending order
    for (int w = threadIdx.x; w < words; w += blockDim.x) {
      uint32_t bits = bm[w];
      uint32_t k = pre[w];
      while (bits) {
        int b = __ffs(bits) - 1;
        bits &= bits - 1;
        bidx[base + k++] = lo + (w << 5) + b;
      }
    }
    // zero the block row's value region (contiguous: its blocks are
    // consecutive), then scatter the entries over it — no separate memset
    // pass over the whole value array, and the region is L2-hot for the
    // scatter
    {
      const int64_t v0 = (int64_t)base * rb * cb, v1 = (int64_t)__ldg(blk_ptr + br + 1) * rb * cb;
      constexpr int kPer16 = 16 / (int)sizeof(T);
      const int64_t a0 = (v0 + kPer16 - 1) / kPer16 * kPer16, a1 = v1 / kPer16 * kPer16;
      for (int64_t q = v0 + threadIdx.x; q < min(a0, v1); q += blockDim.x) bval[q] = to_val<T>(0.f);
      for (int64_t q = a0 / kPer16 + threadIdx.x; q < a1 / kPer16; q += blockDim.x)
        reinterpret_cast<uint4*>(bval)[q] = make_uint4(0u, 0u, 0u, 0u);
      for (int64_t q = max(a1, a0) + threadIdx.x; q < v1; q += blockDim.x) bval[q] = to_val<T>(0.f);
    }
    __syncthreads();
    // scatter the entries into their dense blocks
    for (int32_t k = s + threadIdx.x; k < e; k += blockDim.x) {
      int cc = __ldg(col + k), rr = __ldg(row + k);
      const int bq = divp(cc, c, cs);
      int b = bq - lo;
      uint32_t rank = pre[b >> 5] + __popc(bm[b >> 5] & ((1u << (b & 31)) - 1u));
      int64_t blk = (int64_t)base + rank;
      int i = rr - br * r, j = cc - bq * c;
      bval[(blk * rb + i) * cb + j] = to_val<T>(__ldg(val + k));
    }
    __syncthreads();
  }
}

}  // namespace

void scan_counts(sfg_context* ctx, const int32_t* cnt, int64_t n, int32_t* ptr) {
  int tiles = (int)ceil_div(n, kTile);
  auto* status = lookback_status(ctx, tiles);
  SFG_LAUNCH(k_scan_i32, tiles, kBlock, 0, ctx->stream, cnt, (int32_t)n, ptr, status, ctx->epoch++);
}

sfg_tensor* coo_to_bcsr(sfg_context* ctx, const sfg_tensor* s, int64_t r, int64_t c, int dtype) {
  const int64_t m = s->m, n = s->n, nnz = s->nnz;
  sfg_tensor* t = new_tensor(ctx, SFG_BCSR, m, n);
  t->dtype = dtype;
  t->br = r;
  t->bc = c;
  t->nbr = (m - 1) / r + 1;
  t->nbc = (n - 1) / c + 1;
  t->rb = t->nbr == 1 ? m : r;  // one-tile bounds (operators.hpp:275-278)
  t->cb = t->nbc == 1 ? n : c;
  const int32_t nbr = (int32_t)t->nbr;
  int32_t* bptr = dalloc_n<int32_t>(ctx, nbr + 1);
  int32_t* cnt = dalloc_n<int32_t>(ctx, nbr);
  t->ptr = dalloc_n<int32_t>(ctx, nbr + 1);
  if (nnz == 0) {
    SFG_CUDA(cudaMemsetAsync(t->ptr, 0, (nbr + 1) * sizeof(int32_t), ctx->stream));
    t->idx = dalloc_n<int32_t>(ctx, 0);
    t->val = dalloc(ctx, 4);
    dfree(ctx, bptr);
    dfree(ctx, cnt);
    return t;
  }
  SFG_LAUNCH(k_brow_ptr, stream_grid(ctx, ceil_div(nnz, 128 * kBrowVec), kBlock / 32, 1, 8), kBlock, 0,
             ctx->stream, s->row, nnz, (int32_t)r, nbr, bptr);
  int tiles = (int)ceil_div(nbr, kTile);
  auto* status = lookback_status(ctx, tiles);
  const size_t smem_count = kMaxWords * 4;
  const size_t smem_fill = kMaxWords * 8;
  // the attribute is per device (and the call is cheap): set on every call
  SFG_CUDA(cudaFuncSetAttribute(k_count_blocks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_count));
  SFG_CUDA(cudaFuncSetAttribute(k_fill_blocks<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem_fill));
  SFG_CUDA(cudaFuncSetAttribute(k_fill_blocks<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem_fill));
  // bitmap words actually needed: the widest possible row span
  int64_t words = (t->nbc + 31) / 32;
  if (words * 8 > (int64_t)smem_fill)
    raise(SFG_ERR_INVALID_OPERATION,
          "BCSR: block-column range wider than the device bitmap (" + std::to_string(t->nbc) +
              " block columns)");
  int grid = (int)std::min<int64_t>(nbr, (int64_t)ctx->sms * 8);
  // full-range bitmaps (narrow block grids) are kept for the fill kernel
  // when they are small, saving it a second pass over the columns
  uint32_t* gbm = t->nbc <= kFullRangeCols && (int64_t)nbr * words * 4 <= (int64_t(256) << 20)
                      ? dalloc_n<uint32_t>(ctx, (int64_t)nbr * words)
                      : nullptr;
  // half-size CTAs, twice as many resident: one wave over the block rows
  // of a 2,048-block-row matrix instead of 1.7
  const int cgrid = (int)std::min<int64_t>(nbr, (int64_t)ctx->sms * 16);
  SFG_LAUNCH(k_count_blocks, cgrid, kBlock / 2, words * 4, ctx->stream, bptr, s->idx, (int32_t)c, nbr,
             (int32_t)t->nbc, gbm, cnt);
  SFG_LAUNCH(k_scan_i32, tiles, kBlock, 0, ctx->stream, cnt, nbr, t->ptr, status, ctx->epoch++);
  int32_t nblocks = 0;
  read_back(ctx, t->ptr + nbr, sizeof nblocks, &nblocks);
  t->nnz = nblocks;
  int64_t nvals = (int64_t)nblocks * t->rb * t->cb;
  size_t esz = dtype == SFG_BF16 ? 2 : 4;
  t->idx = dalloc_n<int32_t>(ctx, nblocks);
  t->val = dalloc(ctx, nvals * esz);  // zero-filled block row by block row by the fill kernel
  if (dtype == SFG_BF16)
    SFG_LAUNCH(k_fill_blocks<__nv_bfloat16>, grid, kBlock, words * 8, ctx->stream, bptr, s->row,
               s->idx, static_cast<const float*>(s->val), (int32_t)r, (int32_t)c, (int32_t)t->rb,
               (int32_t)t->cb, nbr, (int32_t)t->nbc, gbm, t->ptr, t->idx, static_cast<__nv_bfloat16*>(t->val));
  else
    SFG_LAUNCH(k_fill_blocks<float>, grid, kBlock, words * 8, ctx->stream, bptr, s->row, s->idx,
               static_cast<const float*>(s->val), (int32_t)r, (int32_t)c, (int32_t)t->rb,
               (int32_t)t->cb, nbr, (int32_t)t->nbc, gbm, t->ptr, t->idx, static_cast<float*>(t->val));
  dfree(ctx, gbm);
  dfree(ctx, bptr);
  dfree(ctx, cnt);
  return t;
}

bool block_nz_flags(sfg_context* ctx, const sfg_tensor* s, int64_t r, int64_t c, int64_t min_sum, uint8_t* flag) {
  const int64_t nbr = ceil_div(s->m, r), nbc = ceil_div(s->n, c);
  if (nbc > kDecCounters || nbr >= INT32_MAX) return false;
  if (s->nnz == 0) return true;
  int32_t* bptr = dalloc_n<int32_t>(ctx, nbr + 1);
  SFG_LAUNCH(k_brow_ptr, stream_grid(ctx, ceil_div(s->nnz, 128 * kBrowVec), kBlock / 32, 1, 8), kBlock, 0,
             ctx->stream, s->row, s->nnz, (int32_t)r, (int32_t)nbr, bptr);
  const size_t smem = (size_t)nbc * 4;
  SFG_CUDA(cudaFuncSetAttribute(k_block_nz_flags, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  SFG_LAUNCH(k_block_nz_flags, (int)std::min<int64_t>(nbr, (int64_t)ctx->sms * 16), kBlock, smem, ctx->stream, bptr,
             s->idx, static_cast<const float*>(s->val), (int32_t)c, (int32_t)nbr, (int32_t)nbc, min_sum,
             s->has_zeros != 0, flag);
  dfree(ctx, bptr);
  return true;
}

}  // namespace sfg
