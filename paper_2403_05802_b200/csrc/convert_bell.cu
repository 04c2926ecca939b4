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
