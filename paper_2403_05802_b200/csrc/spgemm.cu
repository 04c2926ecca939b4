// spgemm.cu — two sparse operands:
// run_kernel(spgemm_kernel(), {A, B}) (kernel.hpp:53, 424-567): C[i][j] +=
// A[i][k] B[k][j] into a dense C, like the reference (its run_kernel
// returns a DenseTensor).
//
// Both operands are brought to CSR on the device (the conversions of
// convert_src.cu / the COO paths; zero-valued entries they trim contribute
// nothing), then a warp per row i of A walks its entries (k, a_ik) in order
// and its lanes stream B's row k: C[i][j] += a_ik * b_kj with plain
// read-modify-writes — the columns of one B row are distinct and the k are
// visited one after another, so no two lanes ever touch the same C word
// at once (the reference's co-iterate mode, kernel.hpp:440-488, in
// parallel over rows). fp32 accumulate; tolerance as for SpMM.
#include <algorithm>

#include "devutil.cuh"
#include "internal.cuh"

namespace sfg {

namespace {

constexpr int kBlock = 256;

__global__ void __launch_bounds__(kBlock) k_spgemm_rows(const int32_t* __restrict__ aptr,
                                                         const int32_t* __restrict__ aidx,
                                                         const float* __restrict__ aval, int64_t m,
                                                         const int32_t* __restrict__ bptr,
                                                         const int32_t* __restrict__ bidx,
                                                         const float* __restrict__ bval, float* __restrict__ c,
                                                         int64_t ldc) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < m; i += warps) {
    float* crow = c + i * ldc;
    const int32_t s = __ldg(aptr + i), e = __ldg(aptr + i + 1);
    for (int32_t base = s; base < e; base += 32) {
      const int32_t p = base + lane;
      const int32_t mk = p < e ? __ldg(aidx + p) : 0;
      const float mv = p < e ? __ldg(aval + p) : 0.f;
      const int cnt = min(32, e - base);
      for (int t = 0; t < cnt; ++t) {
        const int32_t k = __shfl_sync(kFull, mk, t);
        const float a = __shfl_sync(kFull, mv, t);
        const int32_t bs = __ldg(bptr + k), be = __ldg(bptr + k + 1);
        for (int32_t q = bs + lane; q < be; q += 32) {
          const int32_t j = __ldg(bidx + q);
          crow[j] = fmaf(a, __ldg(bval + q), crow[j]);
        }
        __syncwarp();  // the next k may write the same columns
      }
    }
  }
}

sfg_tensor* to_csr(sfg_context* ctx, const sfg_tensor* t) {
  sfg_format f{};
  f.kind = SFG_CSR;
  f.value_dtype = SFG_F32;
  if (t->kind == SFG_COO) return coo_to_csr(ctx, t);
  if (t->kind == SFG_DIA || t->kind == SFG_DIAV || t->kind == SFG_BDIA || t->kind == SFG_CSB ||
      t->kind == SFG_C2SR || t->kind == SFG_DCSC || t->kind == SFG_CISR || t->kind == SFG_CISRP) {  // bounds aside
    sfg_tensor* coo = t->kind == SFG_DIA || t->kind == SFG_DIAV     ? dia_to_coo(ctx, t)
                      : t->kind == SFG_DCSC                          ? dcsc_to_coo(ctx, t)
                      : t->kind == SFG_CISR || t->kind == SFG_CISRP ? cisr_to_coo(ctx, t)
                      : t->kind == SFG_BDIA ? bdia_to_coo(ctx, t)
                      : t->kind == SFG_C2SR ? c2sr_to_coo(ctx, t)
                                            : csb_to_coo(ctx, t);
    sfg_tensor* csr = coo_to_csr(ctx, coo);
    free_tensor_arrays(coo);
    delete coo;
    return csr;
  }
  if (t->kind == SFG_ELL || t->kind == SFG_BELL) {  // zero slots add nothing to a product
    sfg_tensor* coo = ell_nonzeros_to_coo(ctx, t);
    sfg_tensor* csr = coo_to_csr(ctx, coo);
    free_tensor_arrays(coo);
    delete coo;
    return csr;
  }
  if (t->kind == SFG_DOK || t->kind == SFG_LIL) {  // the layout is storage only: same entries
    sfg_tensor* soa = aos_to_soa(ctx, t);
    if (soa->kind == SFG_CSR) return soa;
    sfg_tensor* csr = coo_to_csr(ctx, soa);
    free_tensor_arrays(soa);
    delete soa;
    return csr;
  }
  return convert_from_compressed(ctx, t, f);
}

}  // namespace

void spgemm(sfg_context* ctx, const sfg_tensor* a, const sfg_tensor* b, float* c, int64_t ldc, bool accumulate) {
  if (a->n != b->m) raise(SFG_ERR_INVALID_OPERATION, "spgemm: inner extents differ");
  // hybrid operands: the sum of their two parts' products (the reference
  // runs the kernel once per part)
  if (a->kind == SFG_HYB || a->kind == SFG_HBELL) {
    spgemm(ctx, a->part[0], b, c, ldc, accumulate);
    spgemm(ctx, a->part[1], b, c, ldc, true);
    return;
  }
  if (b->kind == SFG_HYB || b->kind == SFG_HBELL) {
    spgemm(ctx, a, b->part[0], c, ldc, accumulate);
    spgemm(ctx, a, b->part[1], c, ldc, true);
    return;
  }
  const int64_t m = a->m, n = b->n;
  if (!accumulate && m > 0 && n > 0) {
    if (ldc == n)
      SFG_CUDA(cudaMemsetAsync(c, 0, m * n * sizeof(float), ctx->stream));
    else
      SFG_CUDA(cudaMemset2DAsync(c, ldc * sizeof(float), 0, n * sizeof(float), m, ctx->stream));
  }
  if (m == 0 || n == 0 || a->nnz == 0 || b->nnz == 0) return;
  sfg_tensor* ac = a->kind == SFG_CSR && a->dtype == SFG_F32 ? nullptr : to_csr(ctx, a);
  sfg_tensor* bc = nullptr;
  try {
    bc = b->kind == SFG_CSR && b->dtype == SFG_F32 ? nullptr : to_csr(ctx, b);
  } catch (...) {
    if (ac) {
      free_tensor_arrays(ac);
      delete ac;
    }
    throw;
  }
  const sfg_tensor* A = ac ? ac : a;
  const sfg_tensor* B = bc ? bc : b;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(m, kBlock / 32), (int64_t)ctx->sms * 16));
  // a BCSR operand comes back over its whole block grid: its extra rows and
  // columns hold no entries, so the logical m bounds the walk
  SFG_LAUNCH(k_spgemm_rows, grid, kBlock, 0, ctx->stream, A->ptr, A->idx, static_cast<const float*>(A->val), m,
             B->ptr, B->idx, static_cast<const float*>(B->val), c, ldc);
  for (sfg_tensor* t : {ac, bc})
    if (t) {
      free_tensor_arrays(t);
      delete t;
    }
}

}  // namespace sfg
