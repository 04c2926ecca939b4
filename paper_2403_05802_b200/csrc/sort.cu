// sort.cu — from_coo on the device: range check, stable LSD radix sort of
// packed (row, col) keys, duplicate rejection or f64 summation.
//
// Reference: from_coo (tensor.hpp:118-162) = range check (131-135), stable
// lexicographic sort_entries (98-114, std::stable_sort), duplicates ->
// DuplicateCoordinate (147-153) or summed in sorted order (154).
//
// Radix sort: one-sweep LSD with 8-bit digits. An upfront pass histograms
// every digit position; each sort pass then streams tiles of 4096 keys:
// per-warp match_any ranking (stable: rounds of 32 consecutive keys in
// input order), per-digit decoupled look-back across tiles for the tile's
// digit offsets, then the tile is ordered by digit in shared memory and
// written out run by run (coalesced, unlike a scatter straight from
// registers, which spreads every warp store over up to 32 digit runs). Digit positions where every key has the same
// digit are skipped.
#include <cuda_bf16.h>

#include <vector>

#include "async.cuh"
#include "devutil.cuh"
#include "internal.cuh"

namespace sfg {

namespace {

constexpr int kBlock = 256;
constexpr int kWarps = kBlock / 32;
constexpr int kRounds = 16;                       // keys per lane
constexpr int kTile = kBlock * kRounds;           // 4096 keys per tile
constexpr int kMaxPasses = 8;

__global__ void __launch_bounds__(kBlock) k_global_hist(const uint64_t* __restrict__ keys, int64_t n,
                                                         int passes, uint32_t* __restrict__ hist) {
  __shared__ uint32_t h[kMaxPasses][256];
  for (int i = threadIdx.x; i < kMaxPasses * 256; i += blockDim.x) (&h[0][0])[i] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k = keys[i];
    for (int p = 0; p < passes; ++p) atomicAdd(&h[p][(k >> (8 * p)) & 0xff], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * 256; i += blockDim.x) {
    uint32_t v = (&h[0][0])[i];
    if (v) atomicAdd(hist + i, v);
  }
}

constexpr int kStageBytes = kTile * 8;  // the tile's keys, ordered by digit
constexpr int kPayInBytes = kTile * 4;  // the tile's payload, input order

template <bool kPayload>
constexpr int onesweep_dyn_smem() {
  return kStageBytes + (kPayload ? kPayInBytes : 0);
}

template <bool kPayload>
__global__ void __launch_bounds__(kBlock, 3) k_onesweep(const uint64_t* __restrict__ kin,
                                                      const uint32_t* __restrict__ pin,
                                                      uint64_t* __restrict__ kout,
                                                      uint32_t* __restrict__ pout, int64_t n,
                                                      int shift, const uint32_t* __restrict__ goff,
                                                      unsigned long long* __restrict__ status,
                                                      uint32_t epoch) {
  static_assert(kBlock == 256, "one thread per digit");
  __shared__ uint32_t wcnt[kWarps][256];
  __shared__ uint32_t dstart[256];  // tile-local start of each digit's run
  __shared__ uint32_t gshift[256];  // output position - tile-local position
  __shared__ uint32_t scan_smem[34];
  extern __shared__ __align__(16) uint8_t dyn[];
  uint64_t* stage = reinterpret_cast<uint64_t*>(dyn);
  uint32_t* pay_in = reinterpret_cast<uint32_t*>(dyn + kStageBytes);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tile = blockIdx.x;
  const int64_t rem = n - (int64_t)tile * kTile;
  const int tn = rem < kTile ? (int)rem : kTile;
  if (kPayload) {
    // the payload goes straight to shared memory, off the register file,
    // while the keys are ranked
    const uint32_t* src = pin + (int64_t)tile * kTile;
    if (tn == kTile) {
#pragma unroll
      for (int c = threadIdx.x; c < kTile / 4; c += kBlock) cp_async16(pay_in + 4 * c, src + 4 * c);
      cp_async_commit();
    } else {
      for (int i = threadIdx.x; i < tn; i += kBlock) pay_in[i] = src[i];
    }
  }
  for (int i = threadIdx.x; i < kWarps * 256; i += blockDim.x) (&wcnt[0][0])[i] = 0;
  __syncthreads();

  const int64_t wbase = (int64_t)tile * kTile + (int64_t)warp * (32 * kRounds);
  uint64_t key[kRounds];
  uint32_t rank[kRounds];
#pragma unroll
  for (int j = 0; j < kRounds; ++j) {
    int64_t i = wbase + j * 32 + lane;
    key[j] = i < n ? kin[i] : 0;
  }
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int j = 0; j < kRounds; ++j) {
    int64_t i = wbase + j * 32 + lane;
    uint32_t d = i < n ? (uint32_t)((key[j] >> shift) & 0xff) : 256u;
    unsigned peers = __match_any_sync(kFull, d);
    int leader = __ffs(peers) - 1;
    uint32_t b = 0;
    if (lane == leader && d < 256) {
      b = wcnt[warp][d];
      wcnt[warp][d] = b + __popc(peers);
    }
    b = __shfl_sync(kFull, b, leader);
    rank[j] = b + __popc(peers & lt);
    __syncwarp();
  }
  __syncthreads();
  // per digit: exclusive prefix over warps, tile total (posted at once so
  // later tiles can proceed), tile-local digit starts, global look-back
  {
    const int d = threadIdx.x;
    uint32_t s = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      uint32_t c = wcnt[w][d];
      wcnt[w][d] = s;
      s += c;
    }
    unsigned long long* st = status + (size_t)tile * 256 + d;
    st_relaxed(st, lb_pack(epoch, tile == 0 ? 2 : 1, s));
    uint32_t tot;
    const uint32_t ds = block_exclusive_scan<uint32_t, kBlock>(s, scan_smem, &tot);
    dstart[d] = ds;
    const uint32_t ep = epoch & 0x3fffffffu;
    uint32_t excl = 0;
    if (tile > 0) {
      // kLook predecessors' words in flight at once: a walk over tiles that
      // have posted only their aggregate costs one L2 round trip per kLook
      // tiles instead of per tile
      constexpr int kLook = 4;
      int t = tile - 1;
      for (bool done = false; !done;) {
        unsigned long long w[kLook];
#pragma unroll
        for (int q = 0; q < kLook; ++q)
          w[q] = t - q >= 0 ? ld_relaxed(status + (size_t)(t - q) * 256 + d) : lb_pack(epoch, 2, 0);
        int q = 0;
        for (; q < kLook; ++q) {
          const uint32_t hi = (uint32_t)(w[q] >> 32);
          const uint32_t state = (hi >> 2) == ep ? (hi & 3u) : 0u;
          if (state == 0) break;  // not posted yet: poll again from here
          excl += (uint32_t)w[q];
          if (state == 2) {
            done = true;
            break;
          }
        }
        t -= q;
      }
      st_relaxed(st, lb_pack(epoch, 2, excl + s));
    }
    gshift[d] = goff[d] + excl - ds;
  }
  __syncthreads();
  // order the tile by digit in shared memory ...
#pragma unroll
  for (int j = 0; j < kRounds; ++j) {
    int64_t i = wbase + j * 32 + lane;
    if (i < n) {
      uint32_t d = (uint32_t)((key[j] >> shift) & 0xff);
      rank[j] += dstart[d] + wcnt[warp][d];
      stage[rank[j]] = key[j];
    }
  }
  __syncthreads();
  // ... then write it out: consecutive threads store consecutive keys of
  // each digit's run
  uint32_t o[kRounds];
#pragma unroll
  for (int r = 0; r < kRounds; ++r) {
    const int i = r * kBlock + threadIdx.x;
    if (i < tn) {
      const uint64_t k = stage[i];
      o[r] = gshift[(k >> shift) & 0xff] + i;
      kout[o[r]] = k;
    }
  }
  if (kPayload) {
    cp_async_wait_all();
    __syncthreads();
    uint32_t* sp = reinterpret_cast<uint32_t*>(stage);
#pragma unroll
    for (int j = 0; j < kRounds; ++j) {
      const int t = warp * (32 * kRounds) + j * 32 + lane;
      if (t < tn) sp[rank[j]] = pay_in[t];
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
      const int i = r * kBlock + threadIdx.x;
      if (i < tn) pout[o[r]] = sp[i];
    }
  }
}

__global__ void k_digit_offsets(uint32_t* __restrict__ hist, int passes) {
  // one warp per pass: exclusive scan of 256 counts, in place
  int p = blockIdx.x;
  if (p >= passes) return;
  uint32_t* h = hist + p * 256;
  int lane = threadIdx.x;
  uint32_t run = 0;
  for (int c = 0; c < 256; c += 32) {
    uint32_t v = h[c + lane];
    uint32_t inc = warp_inclusive_scan(v);
    h[c + lane] = run + inc - v;
    run += __shfl_sync(kFull, inc, 31);
  }
}

// Head flags of sorted keys -> compaction positions (exclusive scan).
constexpr int kUItems = 16;
constexpr int kUTile = kBlock * kUItems;

// Warp-striped: element wbase + 32 j + lane; head flags by ballot, so loads
// and position stores stay coalesced.
__global__ void __launch_bounds__(kBlock) k_unique_pos(const uint64_t* __restrict__ keys, int64_t n,
                                                        int32_t* __restrict__ pos,
                                                        unsigned long long* __restrict__ status,
                                                        uint32_t epoch, int32_t* __restrict__ total,
                                                        unsigned long long* __restrict__ first_dup) {
  __shared__ uint32_t smem[34];
  __shared__ uint32_t slot;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t wbase = (int64_t)blockIdx.x * kUTile + (int64_t)warp * (32 * kUItems);
  uint64_t k[kUItems];
#pragma unroll
  for (int j = 0; j < kUItems; ++j) {
    const int64_t e = wbase + j * 32 + lane;
    k[j] = e < n ? keys[e] : 0;
  }
  const uint64_t before = lane == 0 && wbase > 0 && wbase < n ? keys[wbase - 1] : 0;
  unsigned ball[kUItems];
  uint32_t cnt = 0;
  unsigned long long dup = ~0ull;
#pragma unroll
  for (int j = 0; j < kUItems; ++j) {
    const int64_t e = wbase + j * 32 + lane;
    uint64_t p = __shfl_up_sync(kFull, k[j], 1);
    const uint64_t t31 = j > 0 ? __shfl_sync(kFull, k[j - 1], 31) : before;
    if (lane == 0) p = t31;
    const bool valid = e < n;
    const bool h = valid && (e == 0 || k[j] != p);
    if (valid && !h && k[j] < dup) dup = k[j];
    ball[j] = __ballot_sync(kFull, h);
    cnt += __popc(ball[j]);
  }
  // R-MAT draws repeat often: one guarded atomic per warp, not per lane
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long w = __shfl_xor_sync(kFull, dup, o);
    dup = w < dup ? w : dup;
  }
  if (lane == 0 && dup != ~0ull && dup < *(volatile unsigned long long*)first_dup) atomicMin(first_dup, dup);
  uint32_t tot;
  const uint32_t wex = block_exclusive_scan<uint32_t, kBlock>(lane == 0 ? cnt : 0u, smem, &tot);
  const uint32_t wpre = __shfl_sync(kFull, wex, 0);
  const uint32_t tp = lookback_prefix(status, epoch, blockIdx.x, tot, &slot);
  const unsigned lt = (1u << lane) - 1u;
  uint32_t run = tp + wpre;
#pragma unroll
  for (int j = 0; j < kUItems; ++j) {
    const int64_t e = wbase + j * 32 + lane;
    // position of this key's unique slot
    if (e < n) pos[e] = (int32_t)(run + __popc(ball[j] & lt) + ((ball[j] >> lane) & 1u) - 1u);
    run += __popc(ball[j]);
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) *total = (int32_t)(tp + tot);
}

enum { kBadRange = 1, kZeroValue = 2 };

// Also the radix sort's digit histograms (as k_global_hist), while the
// keys are in registers.
__global__ void __launch_bounds__(kBlock) k_make_keys(const int32_t* __restrict__ row,
                                                       const int32_t* __restrict__ col,
                                                       const float* __restrict__ val, int64_t nnz,
                                                       int32_t m, int32_t n, int cbits, int passes,
                                                       uint64_t* __restrict__ keys,
                                                       uint32_t* __restrict__ pay,
                                                       uint32_t* __restrict__ hist,
                                                       int* __restrict__ flags) {
  __shared__ uint32_t h[kMaxPasses][256];
  for (int i = threadIdx.x; i < kMaxPasses * 256; i += blockDim.x) (&h[0][0])[i] = 0;
  __syncthreads();
  int f = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    int r = row[e], c = col[e];
    if (r < 0 || r >= m || c < 0 || c >= n) f |= kBadRange;
    if (val[e] == 0.f) f |= kZeroValue;
    const uint64_t k = ((uint64_t)(uint32_t)r << cbits) | (uint32_t)c;
    keys[e] = k;
    pay[e] = __float_as_uint(val[e]);
    for (int p = 0; p < passes; ++p) atomicAdd(&h[p][(k >> (8 * p)) & 0xff], 1u);
  }
  f = __reduce_or_sync(kFull, f);
  if (f && (threadIdx.x & 31) == 0) atomicOr(flags, f);
  __syncthreads();
  for (int i = threadIdx.x; i < passes * 256; i += blockDim.x) {
    uint32_t v = (&h[0][0])[i];
    if (v) atomicAdd(hist + i, v);
  }
}

// Unique keys -> canonical COO. With sum_duplicates, the head of each run
// adds the run's values in sorted (= stable input) order in f64, like
// `out.values.back() += t.values[e]` over doubles (tensor.hpp:154), and
// rounds once to fp32.
__global__ void __launch_bounds__(kBlock) k_emit_coo(const uint64_t* __restrict__ keys,
                                                      const uint32_t* __restrict__ pay,
                                                      const int32_t* __restrict__ pos, int64_t n,
                                                      int cbits, int32_t* __restrict__ row,
                                                      int32_t* __restrict__ col,
                                                      float* __restrict__ val) {
  const uint64_t cmask = (1ull << cbits) - 1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k = keys[i];
    if (i > 0 && keys[i - 1] == k) continue;
    double s = (double)__uint_as_float(pay[i]);
    for (int64_t j = i + 1; j < n && keys[j] == k; ++j) s += (double)__uint_as_float(pay[j]);
    int32_t o = pos[i];
    row[o] = (int32_t)(k >> cbits);
    col[o] = (int32_t)(k & cmask);
    val[o] = (float)s;
  }
}

// Without sum_duplicates any repeated key is an error, so an accepted
// input has no duplicates and entry i of the sorted keys is entry i of the
// result: emit straight through, recording the smallest repeated key.
__global__ void __launch_bounds__(kBlock) k_emit_distinct(const uint64_t* __restrict__ keys,
                                                           const uint32_t* __restrict__ pay, int64_t n,
                                                           int cbits, int32_t* __restrict__ row,
                                                           int32_t* __restrict__ col, float* __restrict__ val,
                                                           unsigned long long* __restrict__ first_dup) {
  const uint64_t cmask = (1ull << cbits) - 1;
  unsigned long long dup = ~0ull;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = keys[i];
    if (i > 0 && keys[i - 1] == k && k < dup) dup = k;
    row[i] = (int32_t)(k >> cbits);
    col[i] = (int32_t)(k & cmask);
    val[i] = __uint_as_float(pay[i]);
  }
  if (dup != ~0ull) atomicMin(first_dup, dup);
}

int bits_for(int64_t extent) {
  int b = 0;
  while ((int64_t(1) << b) < extent) ++b;
  return b;
}

}  // namespace

// LSD radix sort of (key, payload) by the low `key_bits` bits. The result
// lands in either the input or the alternate buffer; *kres / *pres say which.
void radix_sort(sfg_context* ctx, uint64_t* keys, uint32_t* pay, int64_t n, int key_bits,
                uint64_t** kres, uint32_t** pres, uint64_t** kalt_out, uint32_t** palt_out, uint32_t* hist) {
  int passes = (key_bits + 7) / 8;
  if (passes > kMaxPasses) passes = kMaxPasses;
  uint64_t* kalt = dalloc_n<uint64_t>(ctx, n);
  uint32_t* palt = pay ? dalloc_n<uint32_t>(ctx, n) : nullptr;
  *kalt_out = kalt;
  *palt_out = palt;
  uint64_t* kin = keys;
  uint32_t* pin = pay;
  uint64_t* kout = kalt;
  uint32_t* pout = palt;
  if (n > 1 && passes > 0) {
    int tiles = (int)ceil_div(n, kTile);
    size_t status_bytes = (size_t)tiles * 256 * 8;
    auto* status = lookback_status(ctx, status_bytes / 8);
    if (!hist) {
      hist = static_cast<uint32_t*>(scratch(ctx, kMaxPasses * 256 * 4 + 256));
      SFG_CUDA(cudaMemsetAsync(hist, 0, kMaxPasses * 256 * 4, ctx->stream));
      SFG_LAUNCH(k_global_hist, stream_grid(ctx, n, kBlock, 8, 4), kBlock, 0, ctx->stream, keys, n,
                 passes, hist);
    }
    std::vector<uint32_t> h(passes * 256);
    SFG_CUDA(cudaMemcpyAsync(h.data(), hist, passes * 256 * 4, cudaMemcpyDeviceToHost, ctx->stream));
    SFG_LAUNCH(k_digit_offsets, passes, 32, 0, ctx->stream, hist, passes);
    SFG_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int p = 0; p < passes; ++p) {
      bool constant = false;
      for (int d = 0; d < 256; ++d) constant |= (h[p * 256 + d] == (uint32_t)n);
      if (constant) continue;
      if (pay) {
        SFG_CUDA(cudaFuncSetAttribute(k_onesweep<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      onesweep_dyn_smem<true>()));
        SFG_LAUNCH(k_onesweep<true>, tiles, kBlock, onesweep_dyn_smem<true>(), ctx->stream, kin, pin, kout,
                   pout, n, 8 * p, hist + p * 256, status, ctx->epoch++);
      } else {
        SFG_LAUNCH(k_onesweep<false>, tiles, kBlock, onesweep_dyn_smem<false>(), ctx->stream, kin, nullptr,
                   kout, nullptr, n, 8 * p, hist + p * 256, status, ctx->epoch++);
      }
      std::swap(kin, kout);
      std::swap(pin, pout);
    }
  }
  *kres = kin;
  *pres = pin;
}

void sort_u64_keys(sfg_context* ctx, uint64_t* keys, int64_t n, int key_bits, uint64_t** sorted_out) {
  uint64_t *kres, *kalt;
  uint32_t *pres, *palt;
  radix_sort(ctx, keys, nullptr, n, key_bits, &kres, &pres, &kalt, &palt);
  if (kres == keys) dfree(ctx, kalt);
  *sorted_out = kres;
}

int64_t unique_positions(sfg_context* ctx, const uint64_t* keys, int64_t n, int32_t* pos) {
  if (n == 0) return 0;
  int tiles = (int)ceil_div(n, kUTile);
  auto* status = lookback_status(ctx, tiles);
  auto* tail = static_cast<unsigned long long*>(scratch(ctx, 64));
  SFG_CUDA(cudaMemsetAsync(tail, 0xff, 16, ctx->stream));
  SFG_LAUNCH(k_unique_pos, tiles, kBlock, 0, ctx->stream, keys, n, pos, status, ctx->epoch++,
             reinterpret_cast<int32_t*>(tail + 1), tail);
  int32_t total[4];
  read_back(ctx, tail, 16, total);
  return total[2];
}

sfg_tensor* sort_coo(sfg_context* ctx, int64_t m, int64_t n, int64_t nnz, const int32_t* row,
                     const int32_t* col, const float* val, bool sum_duplicates) {
  sfg_tensor* t = new_tensor(ctx, SFG_COO, m, n);
  if (nnz == 0) {
    t->row = dalloc_n<int32_t>(ctx, 0);
    t->idx = dalloc_n<int32_t>(ctx, 0);
    t->val = dalloc_n<float>(ctx, 0);
    return t;
  }
  int cbits = bits_for(n), rbits = bits_for(m);
  uint64_t* keys = dalloc_n<uint64_t>(ctx, nnz);
  uint32_t* pay = dalloc_n<uint32_t>(ctx, nnz);
  const int passes = std::min((cbits + rbits + 7) / 8, kMaxPasses);
  // scratch: the digit histograms radix_sort takes over, then the flags
  auto* hist = static_cast<uint32_t*>(scratch(ctx, kMaxPasses * 256 * 4 + 256));
  int* flags = reinterpret_cast<int*>(hist + kMaxPasses * 256);
  SFG_CUDA(cudaMemsetAsync(hist, 0, kMaxPasses * 256 * 4 + 16, ctx->stream));
  SFG_LAUNCH(k_make_keys, stream_grid(ctx, nnz, kBlock, 4), kBlock, 0, ctx->stream, row, col, val,
             nnz, (int32_t)m, (int32_t)n, cbits, passes, keys, pay, hist, flags);
  int f = 0;
  read_back(ctx, flags, 4, &f);
  if (f & kBadRange) {
    dfree(ctx, keys);
    dfree(ctx, pay);
    delete t;
    raise(SFG_ERR_INVALID_OPERATION, "coordinate out of range");
  }
  uint64_t *kres, *kalt;
  uint32_t *pres, *palt;
  radix_sort(ctx, keys, pay, nnz, cbits + rbits, &kres, &pres, &kalt, &palt, hist);
  auto free_sort = [&] {
    dfree(ctx, keys);
    dfree(ctx, pay);
    dfree(ctx, kalt);
    dfree(ctx, palt);
  };
  auto dup_error = [&](uint64_t k) {
    delete t;
    raise(SFG_ERR_DUPLICATE_COORDINATE,
          "duplicate coordinate (" + std::to_string(k >> cbits) + "," +
              std::to_string(k & ((1ull << cbits) - 1)) + ")");
  };
  if (!sum_duplicates) {
    t->row = dalloc_n<int32_t>(ctx, nnz);
    t->idx = dalloc_n<int32_t>(ctx, nnz);
    t->val = dalloc_n<float>(ctx, nnz);
    auto* dup = static_cast<unsigned long long*>(scratch(ctx, 64));
    SFG_CUDA(cudaMemsetAsync(dup, 0xff, 8, ctx->stream));
    SFG_LAUNCH(k_emit_distinct, stream_grid(ctx, nnz, kBlock, 4), kBlock, 0, ctx->stream, kres, pres, nnz,
               cbits, t->row, t->idx, static_cast<float*>(t->val), dup);
    unsigned long long k = 0;
    read_back(ctx, dup, 8, &k);
    free_sort();
    if (k != ~0ull) {
      free_tensor_arrays(t);
      dup_error(k);
    }
    t->nnz = nnz;
    t->has_zeros = (f & kZeroValue) ? 1 : 0;
    return t;
  }
  int32_t* pos = dalloc_n<int32_t>(ctx, nnz);
  // unique_positions also records the smallest duplicated key
  int tiles = (int)ceil_div(nnz, kUTile);
  auto* status = lookback_status(ctx, tiles);
  auto* tail = static_cast<unsigned long long*>(scratch(ctx, 64));
  SFG_CUDA(cudaMemsetAsync(tail, 0xff, 16, ctx->stream));
  SFG_LAUNCH(k_unique_pos, tiles, kBlock, 0, ctx->stream, kres, nnz, pos, status, ctx->epoch++,
             reinterpret_cast<int32_t*>(tail + 1), tail);
  unsigned long long res[2];
  read_back(ctx, tail, 16, res);
  int64_t uniq = static_cast<int32_t>(res[1] & 0xffffffffu);
  t->nnz = uniq;
  // summed duplicates may cancel to zero: only a duplicate-free input keeps
  // the zero-free guarantee
  t->has_zeros = (f & kZeroValue) ? 1 : (res[0] != ~0ull ? -1 : 0);
  t->row = dalloc_n<int32_t>(ctx, uniq);
  t->idx = dalloc_n<int32_t>(ctx, uniq);
  t->val = dalloc_n<float>(ctx, uniq);
  SFG_LAUNCH(k_emit_coo, stream_grid(ctx, nnz, kBlock, 4), kBlock, 0, ctx->stream, kres, pres, pos,
             nnz, cbits, t->row, t->idx, static_cast<float*>(t->val));
  dfree(ctx, pos);
  free_sort();
  return t;
}

}  // namespace sfg
