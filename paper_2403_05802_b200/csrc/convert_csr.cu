// convert_csr.cu — canonical-COO checks and the row-compressed conversions
// COO -> COO / CSR / DCSR, plus row partitioning and row slicing.
//
// Reference semantics (paths relative to proj/include/sparseforge/):
//   CSR  = plan Fill(0) Merge(0)   (planner.hpp:242-249; operators.hpp:346-391)
//          materialize: L0 size, L1 ptr[m+1] + idx[nnz] (storage.hpp:156-200);
//          empty rows are dangling prefixes -> empty ptr runs.
//   DCSR = plan Merge(0); L0 is fused (one node per distinct row,
//          storage.hpp:142-149), L1 ptr[nnr+1] + idx[nnz].
// The canonical COO handed in is (row, col)-sorted and unique
// (from_coo, tensor.hpp:118-162), so both are pure streaming passes.
#include <vector>

#include <algorithm>

#include "devutil.cuh"
#include "internal.cuh"

namespace sfg {

namespace {

constexpr int kBlock = 256;

// ---------------------------------------------------------------- checks
enum { kBadRange = 1, kDuplicate = 2, kUnsorted = 4, kZeroValue = 8 };

__global__ void __launch_bounds__(kBlock) k_check_canonical(const int32_t* __restrict__ row,
                                                             const int32_t* __restrict__ col,
                                                             const float* __restrict__ val,
                                                             int64_t nnz, int32_t m, int32_t n,
                                                             int* __restrict__ flags) {
  int f = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    int r = row[e], c = col[e];
    if (r < 0 || r >= m || c < 0 || c >= n) f |= kBadRange;
    if (val[e] == 0.f) f |= kZeroValue;  // explicit zeros: recorded, not an error
    if (e > 0) {
      int pr = row[e - 1], pc = col[e - 1];
      if (pr == r && pc == c) f |= kDuplicate;
      else if (pr > r || (pr == r && pc > c)) f |= kUnsorted;
    }
  }
  f = __reduce_or_sync(kFull, f);
  if ((threadIdx.x & 31) == 0 && f) atomicOr(flags, f);
}

// ----------------------------------------------------------- COO -> CSR
// A warp owns chunks of 128*kCsrVec consecutive entries (128-bit
// loads/stores of row, col, val) and writes the row pointers of the rows
// each chunk opens (chunk_row_ptr: ptr[q] = first entry with row >= q).
constexpr int kCsrVec = 2;

__global__ void __launch_bounds__(kBlock) k_coo_to_csr(const int32_t* __restrict__ row,
                                                        const int32_t* __restrict__ col,
                                                        const float* __restrict__ val, int64_t nnz,
                                                        int32_t m, int32_t* __restrict__ ptr,
                                                        int32_t* __restrict__ ocol,
                                                        float* __restrict__ oval) {
  constexpr int kChunk = 128 * kCsrVec;
  __shared__ __align__(16) int32_t s_rows[kBlock / 32][kChunk];
  const int lane = threadIdx.x & 31;
  const int64_t nchunk = (nnz + kChunk - 1) / kChunk;
  const int64_t warps = (int64_t)gridDim.x * (kBlock / 32);
  // a warp per chunk: uniform trip count (chunk_row_ptr is a warp collective)
  for (int64_t ch = (int64_t)blockIdx.x * (kBlock / 32) + (threadIdx.x >> 5); ch < nchunk; ch += warps) {
    const int64_t base = ch * kChunk;
    RowChunk<kCsrVec> c;
    load_row_chunk(row, nnz, base, c);
#pragma unroll
    for (int g = 0; g < kCsrVec; ++g) {
      int64_t e0 = base + 128 * g + 4 * lane;
      if (c.full) {
        int4 cc = ld_stream(reinterpret_cast<const int4*>(col + e0));
        float4 vv = ld_stream(reinterpret_cast<const float4*>(val + e0));
        st_stream(reinterpret_cast<int4*>(ocol + e0), cc);
        st_stream(reinterpret_cast<float4*>(oval + e0), vv);
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (e0 + i < nnz) {
            ocol[e0 + i] = col[e0 + i];
            oval[e0 + i] = val[e0 + i];
          }
      }
    }
    chunk_row_ptr(c, nnz, base, m, s_rows[threadIdx.x >> 5], ptr);
  }
}

// nnz == 0: every row is empty.
__global__ void k_fill_i32(int32_t* __restrict__ p, int64_t n, int32_t v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

// ---------------------------------------------------------- COO -> DCSR
// Row heads (e == 0 or row[e] != row[e-1]) are compacted: tile t learns how
// many heads precede it and writes L0.idx[pos] = row, L1.ptr[pos] = e
// directly. The column and value arrays are the COO's own: the heads
// kernel moves each tile's words with 16-byte loads and stores (one launch
// less than a separate copy: 80 -> 65-71 µs at config 3). (A single-pass decoupled look-back
// version, copies included, took 59 µs on config 3; without the copies
// still 41 µs — the look-back serialised the tiles.)
constexpr int kDcsrItems = 16;  // per lane, warp-striped
constexpr int kDcsrTile = kBlock * kDcsrItems;

// Row heads without a serial look-back: k_dcsr_count counts each tile's
// heads (a tile is one CTA's kDcsrTile entries, warp-striped), then
// k_dcsr_heads has every CTA sum the counts of the tiles before it (at most
// a few thousand words, read once per CTA) and write its heads — two
// streaming passes over the rows that never wait on another CTA.
__device__ __forceinline__ void dcsr_tile_heads(const int32_t* __restrict__ row, int64_t nnz, int64_t wbase,
                                                int (&r)[kDcsrItems], unsigned (&ball)[kDcsrItems], uint32_t& cnt) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < kDcsrItems; ++j) {
    const int64_t e = wbase + 32 * j + lane;
    r[j] = e < nnz ? ld_stream(row + e) : -2;
  }
  const int before = lane == 0 && wbase > 0 && wbase < nnz ? __ldg(row + wbase - 1) : -1;
  cnt = 0;
#pragma unroll
  for (int j = 0; j < kDcsrItems; ++j) {
    const int64_t e = wbase + 32 * j + lane;
    int p = __shfl_up_sync(kFull, r[j], 1);
    const int t31 = j > 0 ? __shfl_sync(kFull, r[j - 1], 31) : before;
    if (lane == 0) p = t31;
    const bool h = e < nnz && (e == 0 || r[j] != p);
    ball[j] = __ballot_sync(kFull, h);
    cnt += __popc(ball[j]);
  }
}

__global__ void __launch_bounds__(kBlock) k_dcsr_count(const int32_t* __restrict__ row, int64_t nnz,
                                                       uint32_t* __restrict__ tile_cnt) {
  __shared__ uint32_t wsum[kBlock / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t wbase = (int64_t)blockIdx.x * kDcsrTile + (int64_t)warp * (32 * kDcsrItems);
  int r[kDcsrItems];
  unsigned ball[kDcsrItems];
  uint32_t cnt;
  dcsr_tile_heads(row, nnz, wbase, r, ball, cnt);
  if (lane == 0) wsum[warp] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < kBlock / 32; ++w) t += wsum[w];
    tile_cnt[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(kBlock) k_dcsr_heads(const int32_t* __restrict__ row, int64_t nnz,
                                                       const uint32_t* __restrict__ tile_cnt,
                                                       int32_t* __restrict__ orow, int32_t* __restrict__ optr,
                                                       int32_t* __restrict__ nnr_out,
                                                       const int4* __restrict__ cin, const int4* __restrict__ vin,
                                                       int4* __restrict__ cout, int4* __restrict__ vout) {
  __shared__ uint32_t smem[34];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tile = blockIdx.x;
  // the tile's column and value words move unchanged (16-byte copies,
  // issued first so they overlap the head detection)
  {
    const int64_t q0 = (int64_t)tile * (kDcsrTile / 4), q1 = min((int64_t)(tile + 1) * (kDcsrTile / 4), nnz / 4);
    for (int64_t q = q0 + threadIdx.x; q < q1; q += kBlock) {
      const int4 a = ld_stream(cin + q), b = ld_stream(vin + q);
      st_stream(cout + q, a);
      st_stream(vout + q, b);
    }
    if (tile == gridDim.x - 1)
      for (int64_t e = (nnz / 4) * 4 + threadIdx.x; e < nnz; e += kBlock) {
        reinterpret_cast<int32_t*>(cout)[e] = reinterpret_cast<const int32_t*>(cin)[e];
        reinterpret_cast<int32_t*>(vout)[e] = reinterpret_cast<const int32_t*>(vin)[e];
      }
  }
  // heads before this tile: the counts of tiles 0 .. tile-1
  uint32_t before = 0;
  for (int i = threadIdx.x; i < tile; i += kBlock) before += __ldg(tile_cnt + i);
  const int64_t wbase = (int64_t)tile * kDcsrTile + (int64_t)warp * (32 * kDcsrItems);
  int r[kDcsrItems];
  unsigned ball[kDcsrItems];
  uint32_t cnt;
  dcsr_tile_heads(row, nnz, wbase, r, ball, cnt);
  // the tile's prefix (the threads' partial sums added up), then this
  // warp's offset inside the tile
  uint32_t tile_prefix;
  block_exclusive_scan<uint32_t, kBlock>(before, smem, &tile_prefix);
  uint32_t wtot;
  const uint32_t wex = block_exclusive_scan<uint32_t, kBlock>(lane == 0 ? cnt : 0u, smem, &wtot);
  uint32_t pos = tile_prefix + __shfl_sync(kFull, wex, 0);
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int j = 0; j < kDcsrItems; ++j) {
    if ((ball[j] >> lane) & 1u) {
      const uint32_t q = pos + __popc(ball[j] & lt);
      orow[q] = r[j];
      optr[q] = (int32_t)(wbase + 32 * j + lane);
    }
    pos += __popc(ball[j]);
  }
  if (tile == gridDim.x - 1 && threadIdx.x == 0) {
    const uint32_t nnr = tile_prefix + wtot;
    optr[nnr] = (int32_t)nnz;
    *nnr_out = (int32_t)nnr;
  }
}

// ------------------------------------------------------- row partitioning
__global__ void k_lower_bound_rows(const int32_t* __restrict__ row, int64_t nnz,
                                   const int64_t* __restrict__ keys, int nkeys,
                                   int64_t* __restrict__ out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nkeys) return;
  int64_t lo = 0, hi = nnz, key = keys[i];
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (row[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  out[i] = lo;
}

__global__ void k_gather_rows(const int32_t* __restrict__ row, const int64_t* __restrict__ pos,
                              int nkeys, int64_t nnz, int32_t m, int64_t* __restrict__ out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nkeys) return;
  out[i] = pos[i] < nnz ? row[pos[i]] : m;
}

__global__ void k_slice_rows(const int32_t* __restrict__ row, const int32_t* __restrict__ col,
                             const float* __restrict__ val, int64_t e0, int64_t count, int32_t r0,
                             int32_t* __restrict__ orow, int32_t* __restrict__ ocol,
                             float* __restrict__ oval) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    orow[i] = row[e0 + i] - r0;
    ocol[i] = col[e0 + i];
    oval[i] = val[e0 + i];
  }
}

}  // namespace

int check_coo_canonical(sfg_context* ctx, const int32_t* row, const int32_t* col, const float* val,
                        int64_t m, int64_t n, int64_t nnz) {
  if (nnz == 0) return 0;
  int* flags = static_cast<int*>(scratch(ctx, 64));
  SFG_CUDA(cudaMemsetAsync(flags, 0, sizeof(int), ctx->stream));
  SFG_LAUNCH(k_check_canonical, stream_grid(ctx, nnz, kBlock, 4), kBlock, 0, ctx->stream, row, col, val,
             nnz, (int32_t)m, (int32_t)n, flags);
  int f = 0;
  read_back(ctx, flags, sizeof f, &f);
  if (f & kBadRange) raise(SFG_ERR_INVALID_OPERATION, "coordinate out of range");
  if (f & kUnsorted)
    raise(SFG_ERR_INVALID_OPERATION, "input flagged SORTED is not (row, col)-sorted");
  if (f & kDuplicate) raise(SFG_ERR_DUPLICATE_COORDINATE, "duplicate coordinate");
  return (f & kZeroValue) ? 1 : 0;
}

sfg_tensor* coo_to_coo(sfg_context* ctx, const sfg_tensor* s) {
  sfg_tensor* t = new_tensor(ctx, SFG_COO, s->m, s->n);
  t->nnz = s->nnz;
  t->has_zeros = s->has_zeros;
  t->row = dalloc_n<int32_t>(ctx, s->nnz);
  t->idx = dalloc_n<int32_t>(ctx, s->nnz);
  t->val = dalloc_n<float>(ctx, s->nnz);
  SFG_CUDA(cudaMemcpyAsync(t->row, s->row, s->nnz * 4, cudaMemcpyDeviceToDevice, ctx->stream));
  SFG_CUDA(cudaMemcpyAsync(t->idx, s->idx, s->nnz * 4, cudaMemcpyDeviceToDevice, ctx->stream));
  SFG_CUDA(cudaMemcpyAsync(t->val, s->val, s->nnz * 4, cudaMemcpyDeviceToDevice, ctx->stream));
  return t;
}

void compress_sorted(sfg_context* ctx, const int32_t* key, const int32_t* other, const float* val,
                     int64_t nnz, int64_t extent, int32_t* ptr, int32_t* oidx, float* oval) {
  if (nnz == 0) {
    SFG_LAUNCH(k_fill_i32, stream_grid(ctx, extent + 1, kBlock, 4), kBlock, 0, ctx->stream, ptr,
               extent + 1, 0);
    return;
  }
  SFG_LAUNCH(k_coo_to_csr, stream_grid(ctx, ceil_div(nnz, 128 * kCsrVec), kBlock / 32, 1, 8), kBlock, 0, ctx->stream,
             key, other, val, nnz, (int32_t)extent, ptr, oidx, oval);
}

sfg_tensor* coo_to_csr(sfg_context* ctx, const sfg_tensor* s) {
  sfg_tensor* t = new_tensor(ctx, SFG_CSR, s->m, s->n);
  t->nnz = s->nnz;
  t->ptr = dalloc_n<int32_t>(ctx, s->m + 1);
  t->idx = dalloc_n<int32_t>(ctx, s->nnz);
  t->val = dalloc_n<float>(ctx, s->nnz);
  if (s->nnz == 0) {
    SFG_LAUNCH(k_fill_i32, stream_grid(ctx, s->m + 1, kBlock, 4), kBlock, 0, ctx->stream, t->ptr,
               s->m + 1, 0);
    return t;
  }
  SFG_LAUNCH(k_coo_to_csr, stream_grid(ctx, ceil_div(s->nnz, 128 * kCsrVec), kBlock / 32, 1, 8), kBlock, 0, ctx->stream, s->row,
             s->idx, static_cast<const float*>(s->val), s->nnz, (int32_t)s->m, t->ptr, t->idx,
             static_cast<float*>(t->val));
  return t;
}

sfg_tensor* coo_to_dcsr(sfg_context* ctx, const sfg_tensor* s) {
  sfg_tensor* t = new_tensor(ctx, SFG_DCSR, s->m, s->n);
  t->nnz = s->nnz;
  int64_t cap = s->nnz < s->m ? s->nnz : s->m;  // nnr <= min(nnz, m)
  t->row = dalloc_n<int32_t>(ctx, cap);
  t->ptr = dalloc_n<int32_t>(ctx, cap + 1);
  t->idx = dalloc_n<int32_t>(ctx, s->nnz);
  t->val = dalloc_n<float>(ctx, s->nnz);
  if (s->nnz == 0) {
    SFG_LAUNCH(k_fill_i32, 1, 32, 0, ctx->stream, t->ptr, 1, 0);
    t->nnr = 0;
    return t;
  }
  int tiles = (int)ceil_div(s->nnz, kDcsrTile);
  auto* sc = static_cast<uint32_t*>(scratch(ctx, 64 + (size_t)tiles * 4));
  int32_t* nnr_dev = reinterpret_cast<int32_t*>(sc);
  uint32_t* tile_cnt = sc + 16;
  SFG_LAUNCH(k_dcsr_count, tiles, kBlock, 0, ctx->stream, s->row, s->nnz, tile_cnt);
  SFG_LAUNCH(k_dcsr_heads, tiles, kBlock, 0, ctx->stream, s->row, s->nnz, tile_cnt, t->row, t->ptr, nnr_dev,
             reinterpret_cast<const int4*>(s->idx), reinterpret_cast<const int4*>(s->val),
             reinterpret_cast<int4*>(t->idx), reinterpret_cast<int4*>(t->val));
  // nnr is read back asynchronously: the tensor is usable at once and the
  // host only waits where the count is needed (tensor_nnr)
  t->nnr_slot = size_slot_start(ctx, nnr_dev);
  if (t->nnr_slot < 0) {
    int32_t nnr = 0;
    read_back(ctx, nnr_dev, sizeof nnr, &nnr);
    t->nnr = nnr;
  }
  return t;
}

// The boundary rule, shared by the device and host entry points: partition
// p starts at the row holding entry floor(p * nnz / P) (nnz balanced to
// within one row), monotone, [0, m]. `row_at(e)` returns the
// row of entry e of the row-sorted COO.
template <class RowAt>
static void bounds_from_quantiles(int64_t m, int64_t nnz, int parts, RowAt row_at, int64_t* bounds) {
  bounds[0] = 0;
  bounds[parts] = m;
  for (int p = 1; p < parts; ++p) {
    int64_t b = nnz == 0 ? m * p / parts : row_at(nnz * p / parts);
    if (b < bounds[p - 1]) b = bounds[p - 1];
    bounds[p] = b;
  }
}

void row_bounds_host(const int32_t* rows, int64_t nnz, int64_t m, int parts, int64_t* bounds) {
  bounds_from_quantiles(m, nnz, parts, [&](int64_t e) -> int64_t { return rows[e]; }, bounds);
}

void row_partition(sfg_context* ctx, const sfg_tensor* coo, int parts, int64_t* bounds) {
  if (parts == 1 || coo->nnz == 0) {
    bounds_from_quantiles(coo->m, coo->nnz, parts, [](int64_t) -> int64_t { return 0; }, bounds);
    return;
  }
  // the P - 1 quantile entries' rows, gathered on the device
  int64_t* dpos = dalloc_n<int64_t>(ctx, parts);
  std::vector<int64_t> pos(parts - 1);
  for (int p = 1; p < parts; ++p) pos[p - 1] = coo->nnz * p / parts;
  SFG_CUDA(cudaMemcpyAsync(dpos, pos.data(), (parts - 1) * 8, cudaMemcpyHostToDevice, ctx->stream));
  int64_t* drows = dalloc_n<int64_t>(ctx, parts);
  SFG_LAUNCH(k_gather_rows, (int)ceil_div(parts - 1, 256), 256, 0, ctx->stream, coo->row, dpos, parts - 1,
             coo->nnz, (int32_t)coo->m, drows);
  std::vector<int64_t> rows(parts - 1);
  SFG_CUDA(cudaMemcpyAsync(rows.data(), drows, (parts - 1) * 8, cudaMemcpyDeviceToHost, ctx->stream));
  SFG_CUDA(cudaStreamSynchronize(ctx->stream));
  dfree(ctx, dpos);
  dfree(ctx, drows);
  bounds_from_quantiles(coo->m, coo->nnz, parts,
                        [&](int64_t e) -> int64_t { return rows[static_cast<size_t>(
                                                       std::lower_bound(pos.begin(), pos.end(), e) - pos.begin())]; },
                        bounds);
}

sfg_tensor* coo_slice_rows(sfg_context* ctx, const sfg_tensor* coo, int64_t r0, int64_t r1) {
  int64_t keys[2] = {r0, r1};
  int64_t* dk = dalloc_n<int64_t>(ctx, 4);
  SFG_CUDA(cudaMemcpyAsync(dk, keys, 16, cudaMemcpyHostToDevice, ctx->stream));
  SFG_LAUNCH(k_lower_bound_rows, 1, 32, 0, ctx->stream, coo->row, coo->nnz, dk, 2, dk + 2);
  int64_t pos[2];
  read_back(ctx, dk + 2, 16, pos);
  dfree(ctx, dk);
  sfg_tensor* t = new_tensor(ctx, SFG_COO, r1 - r0, coo->n);
  int64_t count = pos[1] - pos[0];
  t->nnz = count;
  t->has_zeros = coo->has_zeros == 0 ? 0 : -1;
  t->row = dalloc_n<int32_t>(ctx, count);
  t->idx = dalloc_n<int32_t>(ctx, count);
  t->val = dalloc_n<float>(ctx, count);
  if (count)
    SFG_LAUNCH(k_slice_rows, stream_grid(ctx, count, kBlock, 4), kBlock, 0, ctx->stream, coo->row,
               coo->idx, static_cast<const float*>(coo->val), pos[0], count, (int32_t)r0, t->row,
               t->idx, static_cast<float*>(t->val));
  return t;
}

}  // namespace sfg
