// pack.cu — the value-layout (AoS) formats: Pack(0,1) over COO (DOK) and
// over CSR (LIL).
//
// Reference: Pack(i, j) (operators.hpp:424-430) marks the values and the
// coordinates of levels i..j as one array of structs; materialize carries
// the layout (storage.hpp:128-133) and the container writes its tag
// (io.hpp:262-268). The reference keeps the arrays separate and the tag as
// metadata; here the layout is physical: one record per entry, the level-0
// and level-1 coordinates (DOK: row, col) or the level-1 coordinate (LIL:
// col, the rows being the dense level 0 + ptr) next to the value, so a
// kernel reading an entry touches one contiguous record.
//   DOK: {row, col, val} (12 bytes)      LIL: ptr[m+1] + {col, val} (8 bytes)
// Pack / unpack move 4 entries per thread with 128-bit loads and stores on
// both sides (three / two 16-byte stores of records per four entries).
#include "devutil.cuh"
#include "internal.cuh"

namespace sfg {

namespace {

constexpr int kBlock = 256;

// SoA -> AoS. W = 3 (row, col, val) or 2 (col, val; row == nullptr).
template <int W>
__global__ void __launch_bounds__(kBlock) k_pack(const int32_t* __restrict__ row, const int32_t* __restrict__ col,
                                                 const float* __restrict__ val, int64_t nnz,
                                                 int32_t* __restrict__ rec) {
  const int64_t quads = nnz / 4;
  const bool vec = ((reinterpret_cast<uintptr_t>(col) | reinterpret_cast<uintptr_t>(val) |
                     reinterpret_cast<uintptr_t>(row) | reinterpret_cast<uintptr_t>(rec)) & 15) == 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (vec) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < quads; q += stride) {
      const int4 c = ld_stream(reinterpret_cast<const int4*>(col) + q);
      const float4 v = ld_stream(reinterpret_cast<const float4*>(val) + q);
      int4* out = reinterpret_cast<int4*>(rec + q * 4 * W);
      if constexpr (W == 3) {
        const int4 r = ld_stream(reinterpret_cast<const int4*>(row) + q);
        st_stream(out + 0, make_int4(r.x, c.x, __float_as_int(v.x), r.y));
        st_stream(out + 1, make_int4(c.y, __float_as_int(v.y), r.z, c.z));
        st_stream(out + 2, make_int4(__float_as_int(v.z), r.w, c.w, __float_as_int(v.w)));
      } else {
        st_stream(out + 0, make_int4(c.x, __float_as_int(v.x), c.y, __float_as_int(v.y)));
        st_stream(out + 1, make_int4(c.z, __float_as_int(v.z), c.w, __float_as_int(v.w)));
      }
    }
  }
  for (int64_t e = (vec ? quads * 4 : 0) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += stride) {
    int32_t* out = rec + e * W;
    if constexpr (W == 3) out[0] = row[e];
    out[W - 2] = col[e];
    out[W - 1] = __float_as_int(val[e]);
  }
}

// AoS -> SoA.
template <int W>
__global__ void __launch_bounds__(kBlock) k_unpack(const int32_t* __restrict__ rec, int64_t nnz,
                                                   int32_t* __restrict__ row, int32_t* __restrict__ col,
                                                   float* __restrict__ val) {
  const int64_t quads = nnz / 4;
  const bool vec = ((reinterpret_cast<uintptr_t>(col) | reinterpret_cast<uintptr_t>(val) |
                     reinterpret_cast<uintptr_t>(row) | reinterpret_cast<uintptr_t>(rec)) & 15) == 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (vec) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < quads; q += stride) {
      const int4* in = reinterpret_cast<const int4*>(rec + q * 4 * W);
      if constexpr (W == 3) {
        const int4 a = ld_stream(in), b = ld_stream(in + 1), c = ld_stream(in + 2);
        st_stream(reinterpret_cast<int4*>(row) + q, make_int4(a.x, a.w, b.z, c.y));
        st_stream(reinterpret_cast<int4*>(col) + q, make_int4(a.y, b.x, b.w, c.z));
        st_stream(reinterpret_cast<int4*>(val) + q, make_int4(a.z, b.y, c.x, c.w));
      } else {
        const int4 a = ld_stream(in), b = ld_stream(in + 1);
        st_stream(reinterpret_cast<int4*>(col) + q, make_int4(a.x, a.z, b.x, b.z));
        st_stream(reinterpret_cast<int4*>(val) + q, make_int4(a.y, a.w, b.y, b.w));
      }
    }
  }
  for (int64_t e = (vec ? quads * 4 : 0) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += stride) {
    const int32_t* in = rec + e * W;
    if constexpr (W == 3) row[e] = in[0];
    col[e] = in[W - 2];
    val[e] = __int_as_float(in[W - 1]);
  }
}

int pack_grid(sfg_context* ctx, int64_t nnz) { return stream_grid(ctx, ceil_div(nnz, 4), kBlock, 1, 8); }

}  // namespace

void aos_pack_into(sfg_context* ctx, sfg_tensor* t, const int32_t* row, const int32_t* idx, const float* val) {
  if (t->nnz == 0) return;
  auto* rec = static_cast<int32_t*>(t->val);
  if (t->kind == SFG_DOK)
    SFG_LAUNCH(k_pack<3>, pack_grid(ctx, t->nnz), kBlock, 0, ctx->stream, row, idx, val, t->nnz, rec);
  else
    SFG_LAUNCH(k_pack<2>, pack_grid(ctx, t->nnz), kBlock, 0, ctx->stream, nullptr, idx, val, t->nnz, rec);
}

sfg_tensor* coo_to_dok(sfg_context* ctx, const sfg_tensor* s) {
  // plan: Pack(0,1) — the coordinates and values of the canonical COO, one
  // record per entry in the same (row-sorted) order
  sfg_tensor* t = new_tensor(ctx, SFG_DOK, s->m, s->n);
  t->nnz = s->nnz;
  t->has_zeros = s->has_zeros;
  t->val = dalloc_n<int32_t>(ctx, s->nnz * 3);
  aos_pack_into(ctx, t, s->row, s->idx, static_cast<const float*>(s->val));
  return t;
}

sfg_tensor* coo_to_lil(sfg_context* ctx, const sfg_tensor* s) {
  // plan: Fill(0) Merge(0) Pack(0,1) — the CSR arrays, then the column and
  // value of each entry packed into one record
  sfg_tensor* csr = coo_to_csr(ctx, s);
  sfg_tensor* t = new_tensor(ctx, SFG_LIL, s->m, s->n);
  t->nnz = csr->nnz;
  t->ptr = csr->ptr;
  csr->ptr = nullptr;
  t->val = dalloc_n<int32_t>(ctx, csr->nnz * 2);
  aos_pack_into(ctx, t, nullptr, csr->idx, static_cast<const float*>(csr->val));
  free_tensor_arrays(csr);
  delete csr;
  return t;
}

void aos_unpack(sfg_context* ctx, const sfg_tensor* t, int32_t** row, int32_t** idx, float** val) {
  const bool dok = t->kind == SFG_DOK;
  *row = dok ? dalloc_n<int32_t>(ctx, t->nnz) : nullptr;
  *idx = dalloc_n<int32_t>(ctx, t->nnz);
  *val = dalloc_n<float>(ctx, t->nnz);
  if (t->nnz == 0) return;
  const auto* rec = static_cast<const int32_t*>(t->val);
  if (dok)
    SFG_LAUNCH(k_unpack<3>, pack_grid(ctx, t->nnz), kBlock, 0, ctx->stream, rec, t->nnz, *row, *idx, *val);
  else
    SFG_LAUNCH(k_unpack<2>, pack_grid(ctx, t->nnz), kBlock, 0, ctx->stream, rec, t->nnz, nullptr, *idx, *val);
}

sfg_tensor* aos_to_soa(sfg_context* ctx, const sfg_tensor* t) {
  const bool dok = t->kind == SFG_DOK;
  sfg_tensor* o = new_tensor(ctx, dok ? SFG_COO : SFG_CSR, t->m, t->n);
  o->nnz = t->nnz;
  o->has_zeros = t->has_zeros;
  float* v = nullptr;
  aos_unpack(ctx, t, &o->row, &o->idx, &v);
  o->val = v;
  if (!dok) {
    o->ptr = dalloc_n<int32_t>(ctx, t->m + 1);
    SFG_CUDA(cudaMemcpyAsync(o->ptr, t->ptr, (t->m + 1) * 4, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  return o;
}

}  // namespace sfg
