// convert_bell.cu — COO -> BELL(b), the blocked ELL format.
//
// Reference: BELL(b) = map (d0, d1) -> (indirect(d1/b), d0/b, d1/b, d0%b,
// d1%b) with the block count / slot query chain (formats.hpp:79-85); plan
// TileSplit(0,b) TileSplit(2,b) Swap(1,2) Sum(0) Enumerate(0) Sort Fill(4)
// Fill(3) Fill(1) Vectorize(3) Merge(0). On an input without explicit
// zeros the count query marks every touched b x b block and the slot of a
// block is the ordinal of its block column within its block row
// (query_engine.hpp:166-201), so the materialized arrays
// (storage.hpp:97-234) are the BCSR blocks of each block row laid out slot
// by slot: L0 idx = 0..K-1 (K = most blocks in a block row), L2 idx[K * nbr]
// the block column of (slot, block row), slot-major, and values[K * nbr *
// b * b] the dense blocks in the same order; a block row with fewer blocks
// is padded with block column 0 and a zero block (Fill(1), PadPath).
//
// Device plan: the BCSR conversion (convert_bcsr.cu) gives each block row's
// blocks in block-column order; one relayout pass moves block k of block row
// br to cell (k, br), zero-filling the padding cells. Explicit zeros give
// the slot query its start-offset cases (a block split over several slots),
// which this path does not model: such inputs are rejected.
#include "devutil.cuh"
#include "internal.cuh"

namespace sfg {

namespace {

constexpr int kBlock = 256;

__global__ void k_max_row_blocks(const int32_t* __restrict__ ptr, int64_t nbr, int32_t* __restrict__ out) {
  int m = 0;
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nbr; b += (int64_t)gridDim.x * blockDim.x)
    m = max(m, __ldg(ptr + b + 1) - __ldg(ptr + b));
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

__global__ void k_iota32(int32_t* __restrict__ v, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[i] = (int32_t)i;
}

// A warp per cell (slot k, block row br): block column and the block's
// words (16-byte copies when the block size allows).
__global__ void __launch_bounds__(kBlock) k_bell_fill(const int32_t* __restrict__ ptr,
                                                      const int32_t* __restrict__ bcol,
                                                      const float* __restrict__ bval, int64_t nbr, int64_t k,
                                                      int bsz, int32_t* __restrict__ idx,
                                                      float* __restrict__ val) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t cells = k * nbr;
  const bool vec = (bsz & 3) == 0;
  for (int64_t cell = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; cell < cells; cell += warps) {
    const int64_t slot = cell / nbr, br = cell - slot * nbr;
    const int32_t s = __ldg(ptr + br), e = __ldg(ptr + br + 1);
    const bool real = slot < e - s;
    const int64_t blk = s + slot;
    if (lane == 0) idx[cell] = real ? __ldg(bcol + blk) : 0;
    float* dst = val + cell * bsz;
    const float* src = bval + blk * bsz;
    if (vec) {
      for (int q = lane; q < bsz / 4; q += 32) {
        const float4 w = real ? ld_stream(reinterpret_cast<const float4*>(src) + q) : make_float4(0.f, 0.f, 0.f, 0.f);
        reinterpret_cast<float4*>(dst)[q] = w;
      }
    } else {
      for (int q = lane; q < bsz; q += 32) dst[q] = real ? ld_stream(src + q) : 0.f;
    }
  }
}

__global__ void k_any_zero(const float* __restrict__ val, int64_t n, int* __restrict__ out) {
  bool z = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    z |= ld_stream(val + i) == 0.f;
  if (__any_sync(kFull, z) && (threadIdx.x & 31) == 0) atomicOr(out, 1);
}

}  // namespace

sfg_tensor* coo_to_bell(sfg_context* ctx, const sfg_tensor* s, int64_t b) {
  if (s->has_zeros != 0 && s->nnz) {
    int z = 0;
    auto* flag = static_cast<int*>(scratch(ctx, 64));
    SFG_CUDA(cudaMemsetAsync(flag, 0, 4, ctx->stream));
    SFG_LAUNCH(k_any_zero, stream_grid(ctx, s->nnz, kBlock, 4, 8), kBlock, 0, ctx->stream,
               static_cast<const float*>(s->val), s->nnz, flag);
    read_back(ctx, flag, 4, &z);
    if (z)
      raise(SFG_ERR_UNSUPPORTED_SOURCE,
            "BELL over explicit zeros (the slot query's start offsets split blocks): not held on the device");
  }
  sfg_tensor* bc = coo_to_bcsr(ctx, s, b, b, SFG_F32);
  int32_t kmax = 0;
  if (bc->nbr) {
    auto* mx = static_cast<int32_t*>(scratch(ctx, 64));
    SFG_CUDA(cudaMemsetAsync(mx, 0, 4, ctx->stream));
    SFG_LAUNCH(k_max_row_blocks, (int)std::min<int64_t>(ceil_div(bc->nbr, kBlock), (int64_t)ctx->sms * 8), kBlock,
               0, ctx->stream, bc->ptr, bc->nbr, mx);
    read_back(ctx, mx, 4, &kmax);
  }
  sfg_tensor* t = new_tensor(ctx, SFG_BELL, s->m, s->n);
  t->br = bc->br, t->bc = bc->bc, t->rb = bc->rb, t->cb = bc->cb, t->nbr = bc->nbr, t->nbc = bc->nbc;
  t->k = kmax;
  t->nnz = kmax * bc->nbr;  // cells (slot, block row)
  const int bsz = (int)(bc->rb * bc->cb);
  t->slots = dalloc_n<int32_t>(ctx, kmax);
  t->idx = dalloc_n<int32_t>(ctx, t->nnz);
  t->val = dalloc_n<float>(ctx, t->nnz * bsz);
  if (kmax) {
    SFG_LAUNCH(k_iota32, 1, kBlock, 0, ctx->stream, t->slots, (int64_t)kmax);
    SFG_LAUNCH(k_bell_fill, stream_grid(ctx, t->nnz, kBlock / 32, 1, 16), kBlock, 0, ctx->stream, bc->ptr, bc->idx,
               static_cast<const float*>(bc->val), bc->nbr, (int64_t)kmax, bsz, t->idx, static_cast<float*>(t->val));
  }
  free_tensor_arrays(bc);
  delete bc;
  return t;
}

}  // namespace sfg

// ------------------------------------------------- decompose by blocks
// decompose (decompose.hpp:30-63) with the block count rule
//   sum(value) groupBy (d0, d1) -> (d0/r, d1/c) with value ne 0 -> 1 | otherwise -> 0
// — the paper's hybrid BELL/COO split: the entries of blocks holding at
// least min_sum nonzeros are selected, the rest remain; both parts keep the
// input order. Device: entries keyed (block row, block column·r·c + place in
// block) carry their input index through the canonical radix sort, so each
// block's entries are adjacent; a pass over the sorted keys finds the block
// runs and their nonzero counts and flags every entry at its input index;
// an order-preserving split by the flags (tile counts, scan, scatter) gives
// the two parts.
namespace sfg {
namespace {

__global__ void k_blockdec_keys(const int32_t* __restrict__ row, const int32_t* __restrict__ col, int64_t nnz,
                                int32_t r, int32_t c, int32_t* __restrict__ key, int32_t* __restrict__ sub,
                                float* __restrict__ idx_bits) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t rr = ld_stream(row + e), cc = ld_stream(col + e);
    key[e] = rr / r;
    sub[e] = (int32_t)((int64_t)(cc / c) * r * c + (rr % r) * c + cc % c);
    idx_bits[e] = __int_as_float((int32_t)e);
  }
}

// sorted keys: block runs (same row key, same sub / (r c)) hold <= r c
// entries and the composite (key, sub / (r c)) is nondecreasing, so a thread
// per entry finds its run's ends by binary search inside the r c window
// either side; without explicit zeros the run length is its nonzero count,
// otherwise the run's values are counted.
__global__ void k_blockdec_flags(const int32_t* __restrict__ key, const int32_t* __restrict__ sub,
                                 const float* __restrict__ idx_bits, const float* __restrict__ val_in, int64_t nnz,
                                 int32_t rc, int64_t min_sum, bool count_values, uint8_t* __restrict__ flag) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t k = key[e], b = sub[e] / rc;
    auto same = [&](int64_t q) { return key[q] == k && sub[q] / rc == b; };
    int64_t lo = e - rc + 1 > 0 ? e - rc + 1 : 0, l_hi = e;  // first q in [lo, e] with same(q)
    while (lo < l_hi) {
      const int64_t mid = (lo + l_hi) >> 1;
      if (same(mid)) l_hi = mid; else lo = mid + 1;
    }
    int64_t h_lo = e, hi = e + rc - 1 < nnz - 1 ? e + rc - 1 : nnz - 1;  // last q in [e, hi] with same(q)
    while (h_lo < hi) {
      const int64_t mid = (h_lo + hi + 1) >> 1;
      if (same(mid)) h_lo = mid; else hi = mid - 1;
    }
    int64_t nz = hi - lo + 1;
    if (count_values) {
      nz = 0;
      for (int64_t q = lo; q <= hi; ++q) nz += val_in[__float_as_int(idx_bits[q])] != 0.f ? 1 : 0;
    }
    flag[__float_as_int(idx_bits[e])] = nz >= min_sum ? 1 : 0;
  }
}

constexpr int kSplitItems = 8;
constexpr int kSplitTileF = 256 * kSplitItems;

sfg_tensor* coo_alloc(sfg_context* ctx, int64_t m, int64_t n, int64_t nnz) {
  sfg_tensor* t = new_tensor(ctx, SFG_COO, m, n);
  t->nnz = nnz;
  t->row = dalloc_n<int32_t>(ctx, nnz);
  t->idx = dalloc_n<int32_t>(ctx, nnz);
  t->val = dalloc_n<float>(ctx, nnz);
  return t;
}

__global__ void __launch_bounds__(256) k_flag_count(const uint8_t* __restrict__ flag, int64_t nnz,
                                                    int32_t* __restrict__ cnt) {
  __shared__ int32_t ws[8];
  int32_t n = 0;
  for (int i = 0; i < kSplitItems; ++i) {
    const int64_t e = (int64_t)blockIdx.x * kSplitTileF + i * 256 + threadIdx.x;
    n += e < nnz && flag[e];
  }
  n = warp_sum(n);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = n;
  __syncthreads();
  if (threadIdx.x == 0) {
    int32_t t = 0;
    for (int w = 0; w < 8; ++w) t += ws[w];
    cnt[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(256) k_flag_split(const uint8_t* __restrict__ flag, const int32_t* __restrict__ base,
                                                    const int32_t* __restrict__ row, const int32_t* __restrict__ col,
                                                    const float* __restrict__ val, int64_t nnz,
                                                    int32_t* __restrict__ ar, int32_t* __restrict__ ac,
                                                    float* __restrict__ av, int32_t* __restrict__ br,
                                                    int32_t* __restrict__ bc, float* __restrict__ bv) {
  __shared__ int32_t ws[8];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t t0 = (int64_t)blockIdx.x * kSplitTileF;
  int32_t sel_before = __ldg(base + blockIdx.x);
  for (int i = 0; i < kSplitItems; ++i) {
    const int64_t e = t0 + i * 256 + threadIdx.x;
    const bool in = e < nnz;
    const bool f = in && flag[e];
    const unsigned bal = __ballot_sync(kFull, f);
    if (lane == 0) ws[w] = __popc(bal);
    __syncthreads();
    int32_t wpre = 0, tot = 0;
    for (int q = 0; q < 8; ++q) {
      if (q < w) wpre += ws[q];
      tot += ws[q];
    }
    const int32_t s = sel_before + wpre + __popc(bal & ((1u << lane) - 1u));
    if (in) {
      if (f) {
        ar[s] = row[e], ac[s] = col[e], av[s] = val[e];
      } else {
        const int64_t rpos = e - s;  // entries before e not selected
        br[rpos] = row[e], bc[rpos] = col[e], bv[rpos] = val[e];
      }
    }
    sel_before += tot;
    __syncthreads();
  }
}

}  // namespace

void decompose_blocks(sfg_context* ctx, const sfg_tensor* s, int64_t r, int64_t c, int64_t min_sum,
                      sfg_tensor** sel, sfg_tensor** rem) {
  const int64_t nnz = s->nnz, nbr = ceil_div(s->m, r), nbc = ceil_div(s->n, c);
  if (nbc * r * c >= INT32_MAX) raise(SFG_ERR_INVALID_OPERATION, "decompose by blocks: block keys exceed int32");
  auto* flag = dalloc_n<uint8_t>(ctx, nnz);
  // canonical input with a block-column grid that fits the shared counters:
  // counted in place (convert_bcsr.cu); otherwise the radix path below
  if (!block_nz_flags(ctx, s, r, c, min_sum, flag) && nnz) {
    auto* key = dalloc_n<int32_t>(ctx, nnz);
    auto* sub = dalloc_n<int32_t>(ctx, nnz);
    auto* ib = dalloc_n<float>(ctx, nnz);
    SFG_LAUNCH(k_blockdec_keys, stream_grid(ctx, nnz, kBlock, 4, 8), kBlock, 0, ctx->stream, s->row, s->idx, nnz,
               (int32_t)r, (int32_t)c, key, sub, ib);
    sfg_tensor* sorted = nullptr;
    try {
      sorted = sort_coo(ctx, nbr, nbc * r * c, nnz, key, sub, ib, false);
    } catch (...) {
      for (void* q : {(void*)key, (void*)sub, (void*)ib, (void*)flag}) dfree(ctx, q);
      throw;
    }
    for (void* q : {(void*)key, (void*)sub, (void*)ib}) dfree(ctx, q);
    SFG_LAUNCH(k_blockdec_flags, stream_grid(ctx, nnz, kBlock, 4, 8), kBlock, 0, ctx->stream, sorted->row,
               sorted->idx, static_cast<const float*>(sorted->val), static_cast<const float*>(s->val), nnz,
               (int32_t)(r * c), min_sum, s->has_zeros != 0, flag);
    free_tensor_arrays(sorted);
    delete sorted;
  }
  const int64_t tiles = ceil_div(nnz, (int64_t)kSplitTileF);
  auto* cnt = dalloc_n<int32_t>(ctx, tiles);
  auto* base = dalloc_n<int32_t>(ctx, tiles + 1);
  int32_t nsel = 0;
  if (nnz) {
    SFG_LAUNCH(k_flag_count, (int)tiles, 256, 0, ctx->stream, flag, nnz, cnt);
    scan_counts(ctx, cnt, tiles, base);
    read_back(ctx, base + tiles, 4, &nsel);
  }
  sfg_tensor* a = coo_alloc(ctx, s->m, s->n, nsel);
  sfg_tensor* b = coo_alloc(ctx, s->m, s->n, nnz - nsel);
  a->has_zeros = b->has_zeros = s->has_zeros == 0 ? 0 : -1;
  if (nnz)
    SFG_LAUNCH(k_flag_split, (int)tiles, 256, 0, ctx->stream, flag, base, s->row, s->idx,
               static_cast<const float*>(s->val), nnz, a->row, a->idx, static_cast<float*>(a->val), b->row, b->idx,
               static_cast<float*>(b->val));
  for (void* q : {(void*)flag, (void*)cnt, (void*)base}) dfree(ctx, q);
  *sel = a;
  *rem = b;
}

sfg_tensor* coo_to_hbell(sfg_context* ctx, const sfg_tensor* s, int64_t b, int64_t min_sum) {
  sfg_tensor *sel = nullptr, *rem = nullptr;
  decompose_blocks(ctx, s, b, b, min_sum, &sel, &rem);
  sfg_tensor* h = new_tensor(ctx, SFG_HBELL, s->m, s->n);
  h->threshold = min_sum;
  h->br = h->bc = b;
  try {
    h->part[0] = coo_to_bell(ctx, sel, b);
  } catch (...) {
    for (sfg_tensor* t : {sel, rem}) {
      free_tensor_arrays(t);
      delete t;
    }
    delete h;
    throw;
  }
  free_tensor_arrays(sel);
  delete sel;
  h->part[1] = rem;  // the remainder stays coordinate form (COO)
  return h;
}

}  // namespace sfg
