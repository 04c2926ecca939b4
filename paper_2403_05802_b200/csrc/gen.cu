// gen.cu — seeded synthetic inputs on the device, using the
// same integer generators as the CPU oracle (synth.h), so both sides see
// bit-identical matrices. Bench/test infrastructure, not reference algorithm.
#include "devutil.cuh"
#include "internal.cuh"
#include "synth.h"

namespace sfg {

namespace {

constexpr int kBlock = 256;

// Config 1: row r holds exactly per_row distinct sorted columns.
__global__ void __launch_bounds__(kBlock) k_gen_uniform(uint64_t seed, int32_t m, int32_t n,
                                                         int per_row, int32_t* __restrict__ row,
                                                         int32_t* __restrict__ col,
                                                         float* __restrict__ val) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < m;
       r += (int64_t)gridDim.x * blockDim.x) {
    uint32_t cols[64];
    sfg_uniform_row(seed, (uint32_t)r, (uint32_t)n, per_row, cols);
    int64_t e0 = r * per_row;
    for (int i = 0; i < per_row; ++i) {
      row[e0 + i] = (int32_t)r;
      col[e0 + i] = (int32_t)cols[i];
      val[e0 + i] = sfg_coord_value(seed, (uint32_t)r, cols[i]);
    }
  }
}

__global__ void __launch_bounds__(kBlock) k_gen_keys(uint64_t seed, int kind, int scale, uint32_t m,
                                                      uint32_t n, int64_t draws,
                                                      uint64_t* __restrict__ keys) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < draws;
       e += (int64_t)gridDim.x * blockDim.x)
    keys[e] = kind == 0 ? sfg_rmat_edge(seed, (uint64_t)e, scale)
                        : sfg_uniform_coord(seed, (uint64_t)e, m, n);
}

// Unique sorted keys -> canonical COO with coordinate-hashed values.
__global__ void __launch_bounds__(kBlock) k_keys_to_coo(uint64_t seed,
                                                         const uint64_t* __restrict__ keys,
                                                         const int32_t* __restrict__ pos,
                                                         int64_t n_in, int32_t* __restrict__ row,
                                                         int32_t* __restrict__ col,
                                                         float* __restrict__ val) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_in;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k = keys[i];
    if (i > 0 && keys[i - 1] == k) continue;
    int64_t o = pos[i];
    uint32_t r = (uint32_t)(k >> 32), c = (uint32_t)k;
    row[o] = (int32_t)r;
    col[o] = (int32_t)c;
    val[o] = sfg_coord_value(seed, r, c);
  }
}

__global__ void __launch_bounds__(kBlock) k_gen_dense(uint64_t seed, int64_t count,
                                                       float* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = sfg_dense_value(sfg_hash3(seed, (uint64_t)i, 0x77));
}

}  // namespace

// Defined in sort.cu: head-flag compaction positions of sorted keys.
int64_t unique_positions(sfg_context* ctx, const uint64_t* keys, int64_t n, int32_t* pos);

sfg_tensor* gen_uniform(sfg_context* ctx, uint64_t seed, int64_t m, int64_t n, int per_row) {
  sfg_tensor* t = new_tensor(ctx, SFG_COO, m, n);
  t->nnz = m * per_row;
  t->has_zeros = 0;  // generator values are +-[0.5, 1.5)
  t->row = dalloc_n<int32_t>(ctx, t->nnz);
  t->idx = dalloc_n<int32_t>(ctx, t->nnz);
  t->val = dalloc_n<float>(ctx, t->nnz);
  SFG_LAUNCH(k_gen_uniform, stream_grid(ctx, m, kBlock, 1), kBlock, 0, ctx->stream, seed,
             (int32_t)m, (int32_t)n, per_row, t->row, t->idx, static_cast<float*>(t->val));
  return t;
}

sfg_tensor* gen_from_keys(sfg_context* ctx, uint64_t seed, int kind, int scale, int64_t m,
                          int64_t n, int64_t draws) {
  uint64_t* keys = dalloc_n<uint64_t>(ctx, draws);
  SFG_LAUNCH(k_gen_keys, stream_grid(ctx, draws, kBlock, 4), kBlock, 0, ctx->stream, seed, kind,
             scale, (uint32_t)m, (uint32_t)n, draws, keys);
  int key_bits = 32;
  while (key_bits < 64 && (uint64_t(m - 1) >> (key_bits - 32)) != 0) ++key_bits;
  uint64_t* sorted = nullptr;
  sort_u64_keys(ctx, keys, draws, key_bits, &sorted);
  int32_t* pos = dalloc_n<int32_t>(ctx, draws);
  int64_t u = unique_positions(ctx, sorted, draws, pos);
  sfg_tensor* t = new_tensor(ctx, SFG_COO, m, n);
  t->nnz = u;
  t->has_zeros = 0;
  t->row = dalloc_n<int32_t>(ctx, u);
  t->idx = dalloc_n<int32_t>(ctx, u);
  t->val = dalloc_n<float>(ctx, u);
  SFG_LAUNCH(k_keys_to_coo, stream_grid(ctx, draws, kBlock, 4), kBlock, 0, ctx->stream, seed,
             sorted, pos, draws, t->row, t->idx, static_cast<float*>(t->val));
  dfree(ctx, pos);
  if (sorted != keys) dfree(ctx, sorted);
  dfree(ctx, keys);
  return t;
}

void gen_dense(sfg_context* ctx, uint64_t seed, int64_t count, float* out) {
  if (count <= 0) return;
  SFG_LAUNCH(k_gen_dense, stream_grid(ctx, count, kBlock, 4), kBlock, 0, ctx->stream, seed, count,
             out);
}

}  // namespace sfg
