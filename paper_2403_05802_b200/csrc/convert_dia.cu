// convert_dia.cu — COO -> DIA and COO -> CSB(b) (§8f rank 2, Table-2 formats).
//
// DIA: map (d0, d1) -> (d1 - d0, d0); merge(0), trim(0,0) (formats.hpp:46);
// plan Skew(0,1,-1) Swap(0,1) Sort Fill(1) Vectorize(1) Merge(0). The
// materialized arrays (storage.hpp:97-234): L0 idx = the diagonals d = col -
// row that hold an entry (explicit zeros included), ascending, bounds
// [-(m-1), n-1]; L1 a dense vector over the rows; values[ndiag * m],
// diagonal-major, row i of diagonal d = A[i][i + d] or 0.
// Device: a bitmap of the m + n - 1 diagonals (one bit set per entry),
// ranks by a scan of the bitmap words' popcounts, then the zero-filled value
// panel and one scatter of the entries.
//
// CSB(b): map (d0/b, d1/b, d0%b, d1%b); merge(0,1), trim(2,3)
// (formats.hpp:54-57; r x c blocks, CSB(r) = CSB(r,r)); plan TileSplit(0,r)
// TileSplit(2,c) Swap(1,2) Sort
// Fill(1) Fill(0) Merge(0) Merge(1). Arrays: the dense grid of nbr x nbc
// blocks, L2 ptr[nbr*nbc + 1] (entries per block), L2 idx = the row in the
// block, L3 idx = the column in the block, per entry in (block, row, column)
// order. Device: each entry becomes (block id, r * b + c), the canonical
// radix sort (sort.cu) orders them, the CSR row-pointer pass gives ptr over
// the block grid and one pass splits r / c.
#include "devutil.cuh"
#include "internal.cuh"

namespace sfg {

namespace {

constexpr int kBlock = 256;

__global__ void k_dia_mark(const int32_t* __restrict__ row, const int32_t* __restrict__ col, int64_t nnz,
                           int64_t off, uint32_t* __restrict__ bits) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t d = (int64_t)ld_stream(col + e) - ld_stream(row + e) + off;
    atomicOr(bits + (d >> 5), 1u << (d & 31));
  }
}

// exclusive prefix of the words' popcounts (one CTA; nwords is small:
// (m + n) / 32) and the diagonal list
__global__ void __launch_bounds__(1024) k_dia_ranks(const uint32_t* __restrict__ bits, int64_t nwords, int64_t off,
                                                    int32_t* __restrict__ word_base, int32_t* __restrict__ diags,
                                                    int32_t* __restrict__ ndiag) {
  __shared__ uint32_t sm[34];
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t w0 = 0; w0 < nwords; w0 += 1024) {
    const int64_t w = w0 + threadIdx.x;
    const uint32_t word = w < nwords ? bits[w] : 0u;
    uint32_t tot;
    const uint32_t ex = block_exclusive_scan<uint32_t, 1024>((uint32_t)__popc(word), sm, &tot);
    const uint32_t base = carry + ex;
    if (w < nwords) {
      word_base[w] = (int32_t)base;
      uint32_t b = word, k = base;
      while (b) {
        const int bit = __ffs(b) - 1;
        b &= b - 1;
        diags[k++] = (int32_t)(w * 32 + bit - off);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) *ndiag = (int32_t)carry;
}

// the panel position of an entry: its row (DIA, stride m) or its column
// (DIA-variant, stride n)
__global__ void k_dia_scatter(const int32_t* __restrict__ row, const int32_t* __restrict__ col,
                              const float* __restrict__ val, int64_t nnz, int64_t off, int64_t stride, bool by_col,
                              const uint32_t* __restrict__ bits, const int32_t* __restrict__ word_base,
                              float* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = ld_stream(row + e), c = ld_stream(col + e);
    const int64_t d = (int64_t)c - r + off;
    const uint32_t word = __ldg(bits + (d >> 5));
    const int64_t k = __ldg(word_base + (d >> 5)) + __popc(word & ((1u << (d & 31)) - 1u));
    out[k * stride + (by_col ? c : r)] = ld_stream(val + e);
  }
}

// entry -> (block id, r * b + c) for the CSB sort
__global__ void k_csb_keys(const int32_t* __restrict__ row, const int32_t* __restrict__ col, int64_t nnz, int32_t br,
                           int32_t bc, int64_t nbc, int32_t* __restrict__ key, int32_t* __restrict__ sub) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = ld_stream(row + e), c = ld_stream(col + e);
    key[e] = (int32_t)((int64_t)(r / br) * nbc + c / bc);
    sub[e] = (r % br) * bc + c % bc;
  }
}

__global__ void k_csb_split(const int32_t* __restrict__ sub, int64_t nnz, int32_t bc, int32_t* __restrict__ rin,
                            int32_t* __restrict__ cin) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t q = sub[e];
    rin[e] = q / bc;
    cin[e] = q % bc;
  }
}

// DIA cells holding a nonzero value, as unordered (row, col, val): the
// dematerialization of a DIA source (Devectorize(1) Split(0) Trim(1) drops
// the zero cells — padding and explicit zeros alike)
__global__ void k_dia_nonzeros(const int32_t* __restrict__ diags, const float* __restrict__ val, int64_t ndiag,
                               int64_t m, bool by_col, int32_t* __restrict__ orow, int32_t* __restrict__ ocol,
                               float* __restrict__ oval, unsigned long long* __restrict__ count) {
  const int lane = threadIdx.x & 31;
  const int64_t cells = ndiag * m;  // m: the panel stride (rows, or columns for the variant)
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e - lane < cells;
       e += (int64_t)gridDim.x * blockDim.x) {
    const bool in = e < cells;
    const float v = in ? __ldg(val + e) : 0.f;
    const bool nz = in && v != 0.f;
    const unsigned msk = __ballot_sync(kFull, nz);
    unsigned long long base = 0;
    if (lane == 0 && msk) base = atomicAdd(count, (unsigned long long)__popc(msk));
    base = __shfl_sync(kFull, base, 0);
    if (nz) {
      const int64_t k = e / m, i = e - k * m, d = __ldg(diags + k);
      const unsigned long long at = base + __popc(msk & ((1u << lane) - 1u));
      orow[at] = (int32_t)(by_col ? i - d : i);
      ocol[at] = (int32_t)(by_col ? i : i + d);
      oval[at] = v;
    }
  }
}

// CSB back to canonical COO coordinates (unordered: blocks interleave rows)
__global__ void k_csb_coords(const int32_t* __restrict__ ptr, const int32_t* __restrict__ rin,
                             const int32_t* __restrict__ cin, int64_t nblocks, int64_t nbc, int32_t br, int32_t bc,
                             int32_t* __restrict__ orow, int32_t* __restrict__ ocol) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < nblocks; q += warps) {
    const int64_t r0 = (q / nbc) * br, c0 = (q % nbc) * bc;
    for (int32_t e = __ldg(ptr + q) + lane; e < __ldg(ptr + q + 1); e += 32) {
      orow[e] = (int32_t)(r0 + __ldg(rin + e));
      ocol[e] = (int32_t)(c0 + __ldg(cin + e));
    }
  }
}

}  // namespace

// DIA (variant = false): the dense vector over the rows; DIA-variant: map
// (d0, d1) -> (d1 - d0, d1) (formats.hpp:47-48), the same diagonals with a
// dense vector over the columns: values[ndiag * n], column j of diagonal d =
// A[j - d][j] or 0, L1 bounds [0, n-1].
sfg_tensor* coo_to_dia(sfg_context* ctx, const sfg_tensor* s, bool variant) {
  const int64_t m = s->m, n = s->n, off = m - 1, stride = variant ? n : m;
  const int64_t nd = m + n - 1, nwords = ceil_div(nd, (int64_t)32);
  auto* bits = dalloc_n<uint32_t>(ctx, nwords);
  auto* word_base = dalloc_n<int32_t>(ctx, nwords);
  auto* diags = dalloc_n<int32_t>(ctx, std::min<int64_t>(nd, std::max<int64_t>(s->nnz, 1)));
  auto* nd_dev = static_cast<int32_t*>(scratch(ctx, 64));
  SFG_CUDA(cudaMemsetAsync(bits, 0, nwords * 4, ctx->stream));
  if (s->nnz)
    SFG_LAUNCH(k_dia_mark, stream_grid(ctx, s->nnz, kBlock, 4, 8), kBlock, 0, ctx->stream, s->row, s->idx, s->nnz,
               off, bits);
  SFG_LAUNCH(k_dia_ranks, 1, 1024, 0, ctx->stream, bits, nwords, off, word_base, diags, nd_dev);
  int32_t ndiag = 0;
  read_back(ctx, nd_dev, 4, &ndiag);
  const int64_t cells = (int64_t)ndiag * stride;
  if (cells >= INT32_MAX || cells * 4 > (int64_t)(ctx->total_mem / 2)) {
    for (void* p : {(void*)bits, (void*)word_base, (void*)diags}) dfree(ctx, p);
    raise(SFG_ERR_INVALID_OPERATION, "DIA: " + std::to_string(ndiag) + " diagonals x " + std::to_string(stride) +
                                         (variant ? " columns" : " rows") +
                                         " exceed the device's dense-vector capacity");
  }
  sfg_tensor* t = new_tensor(ctx, variant ? SFG_DIAV : SFG_DIA, m, n);
  t->k = ndiag;
  t->nnz = cells;
  t->slots = diags;  // L0 idx (ascending diagonals)
  t->val = dalloc_n<float>(ctx, cells);
  if (cells) SFG_CUDA(cudaMemsetAsync(t->val, 0, cells * 4, ctx->stream));
  if (s->nnz)
    SFG_LAUNCH(k_dia_scatter, stream_grid(ctx, s->nnz, kBlock, 4, 8), kBlock, 0, ctx->stream, s->row, s->idx,
               static_cast<const float*>(s->val), s->nnz, off, stride, variant, bits, word_base,
               static_cast<float*>(t->val));
  dfree(ctx, bits);
  dfree(ctx, word_base);
  return t;
}

sfg_tensor* coo_to_csb(sfg_context* ctx, const sfg_tensor* s, int64_t br, int64_t bc) {
  const int64_t nbr = ceil_div(s->m, br), nbc = ceil_div(s->n, bc);
  if (nbr * nbc >= INT32_MAX || br * bc >= INT32_MAX)
    raise(SFG_ERR_INVALID_OPERATION, "CSB: the block grid exceeds the int32 index range");
  // entries as (block id, r * b + c), sorted: the CSB order
  auto* key = dalloc_n<int32_t>(ctx, s->nnz);
  auto* sub = dalloc_n<int32_t>(ctx, s->nnz);
  if (s->nnz)
    SFG_LAUNCH(k_csb_keys, stream_grid(ctx, s->nnz, kBlock, 4, 8), kBlock, 0, ctx->stream, s->row, s->idx, s->nnz,
               (int32_t)br, (int32_t)bc, nbc, key, sub);
  sfg_tensor* sorted = nullptr;
  try {
    sorted = sort_coo(ctx, nbr * nbc, br * bc, s->nnz, key, sub, static_cast<const float*>(s->val), false);
  } catch (...) {
    dfree(ctx, key);
    dfree(ctx, sub);
    throw;
  }
  dfree(ctx, key);
  dfree(ctx, sub);
  // ptr over the block grid (the CSR row-pointer pass), then r / c
  sfg_tensor* grid = coo_to_csr(ctx, sorted);
  free_tensor_arrays(sorted);
  delete sorted;
  sfg_tensor* t = new_tensor(ctx, SFG_CSB, s->m, s->n);
  t->br = br, t->bc = bc;
  // in-block extents: the one-tile edge shrinks them (as BCSR's, storage.hpp)
  t->rb = std::min(br, s->m), t->cb = std::min(bc, s->n);
  t->nbr = nbr;
  t->nbc = nbc;
  t->nnz = s->nnz;
  t->ptr = grid->ptr;
  t->val = grid->val;
  t->row = dalloc_n<int32_t>(ctx, s->nnz);  // L2 idx: row in the block
  t->idx = dalloc_n<int32_t>(ctx, s->nnz);  // L3 idx: column in the block
  if (s->nnz)
    SFG_LAUNCH(k_csb_split, stream_grid(ctx, s->nnz, kBlock, 4, 8), kBlock, 0, ctx->stream, grid->idx, s->nnz,
               (int32_t)bc, t->row, t->idx);
  grid->ptr = nullptr;
  grid->val = nullptr;
  free_tensor_arrays(grid);
  delete grid;
  return t;
}

sfg_tensor* csb_to_coo(sfg_context* ctx, const sfg_tensor* t) {
  auto* r = dalloc_n<int32_t>(ctx, t->nnz);
  auto* c = dalloc_n<int32_t>(ctx, t->nnz);
  if (t->nnz)
    SFG_LAUNCH(k_csb_coords, stream_grid(ctx, t->nbr * t->nbc, kBlock / 32, 1, 16), kBlock, 0, ctx->stream, t->ptr,
               t->row, t->idx, t->nbr * t->nbc, t->nbc, (int32_t)t->br, (int32_t)t->bc, r, c);
  sfg_tensor* out = nullptr;
  try {
    out = sort_coo(ctx, t->m, t->n, t->nnz, r, c, static_cast<const float*>(t->val), false);
  } catch (...) {
    dfree(ctx, r);
    dfree(ctx, c);
    throw;
  }
  dfree(ctx, r);
  dfree(ctx, c);
  return out;
}

sfg_tensor* dia_to_coo(sfg_context* ctx, const sfg_tensor* t) {
  const bool by_col = t->kind == SFG_DIAV;
  const int64_t stride = by_col ? t->n : t->m, cells = t->k * stride;
  auto* r = dalloc_n<int32_t>(ctx, cells);
  auto* c = dalloc_n<int32_t>(ctx, cells);
  auto* v = dalloc_n<float>(ctx, cells);
  auto* count = static_cast<unsigned long long*>(scratch(ctx, 64));
  SFG_CUDA(cudaMemsetAsync(count, 0, 8, ctx->stream));
  if (cells)
    SFG_LAUNCH(k_dia_nonzeros, stream_grid(ctx, cells, kBlock, 1, 8), kBlock, 0, ctx->stream, t->slots,
               static_cast<const float*>(t->val), t->k, stride, by_col, r, c, v, count);
  unsigned long long nz = 0;
  read_back(ctx, count, 8, &nz);
  sfg_tensor* out = nullptr;
  try {
    out = sort_coo(ctx, t->m, t->n, (int64_t)nz, r, c, v, false);
  } catch (...) {
    for (void* q : {(void*)r, (void*)c, (void*)v}) dfree(ctx, q);
    throw;
  }
  for (void* q : {(void*)r, (void*)c, (void*)v}) dfree(ctx, q);
  return out;
}

}  // namespace sfg

// --------------------------------------------------------------- BDIA(b)
// BDIA(b): map (d0/b, d1-d0, d0%b); merge(0), trim(1,1) (formats.hpp:74-77);
// plan Skew(0,1,-1) TileSplit(0,b) Swap(1,2) Sort Fill(2) Fill(0)
// Vectorize(2) Merge(0). Arrays: L0 dense over the block rows, L1 ptr[nbr+1]
// + idx = the diagonals d = col - row present in each block row (ascending;
// bounds [-(m-1), n-1]), L2 a dense vector over the rows of the block
// (extent min(b, m)): values[nodes * rb], row r_in of node (block row,
// d) = A[b*br + r_in][b*br + r_in + d] or 0. Device: the canonical radix
// sort orders the entries by (block row, diagonal, row in block) — each
// entry keyed (block row, (d + m - 1) * b + r_in) — then per block row a warp
// counts the distinct diagonals (a ballot of changes), a scan gives ptr, and
// a second warp pass writes idx and scatters the values into the
// zero-filled panel.
namespace sfg {
namespace {

constexpr int kBdiaBlock = 256;

__global__ void k_bdia_keys(const int32_t* __restrict__ row, const int32_t* __restrict__ col, int64_t nnz,
                            int32_t b, int64_t off, int32_t* __restrict__ key, int32_t* __restrict__ sub) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = ld_stream(row + e), c = ld_stream(col + e);
    key[e] = r / b;
    sub[e] = (int32_t)(((int64_t)c - r + off) * b + r % b);
  }
}

// kWrite = false: distinct diagonals per block row into cnt[br];
// kWrite = true: idx[node] = d and the values at node * rb + r_in.
template <bool kWrite>
__global__ void __launch_bounds__(kBdiaBlock) k_bdia_nodes(const int32_t* __restrict__ bptr,
                                                           const int32_t* __restrict__ sub,
                                                           const float* __restrict__ val, int64_t nbr, int32_t b,
                                                           int32_t rb, int64_t off, int32_t* __restrict__ cnt,
                                                           const int32_t* __restrict__ nptr,
                                                           int32_t* __restrict__ idx, float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t br = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; br < nbr; br += warps) {
    const int32_t s = __ldg(bptr + br), e = __ldg(bptr + br + 1);
    int32_t node = kWrite ? __ldg(nptr + br) - 1 : 0;  // the node of the previous entry
    int32_t prev = -1, heads = 0;
    for (int32_t k0 = s; k0 < e; k0 += 32) {
      const int32_t k = k0 + lane;
      const int32_t q = k < e ? __ldg(sub + k) : -1;
      const int32_t d = q >= 0 ? q / b : -1;
      int32_t dp = __shfl_up_sync(kFull, d, 1);
      if (lane == 0) dp = prev;
      const bool head = k < e && d != dp;
      const unsigned hm = __ballot_sync(kFull, head);
      if (kWrite && k < e) {
        const int32_t my = node + __popc(hm & ((2u << lane) - 1u));
        if (head) idx[my] = (int32_t)(d - off);
        out[(int64_t)my * rb + (q - d * b)] = __ldg(val + k);
      }
      node += __popc(hm);
      heads += __popc(hm);
      prev = __shfl_sync(kFull, d, 31);
    }
    if (!kWrite && lane == 0) cnt[br] = heads;
  }
}

}  // namespace

sfg_tensor* coo_to_bdia(sfg_context* ctx, const sfg_tensor* s, int64_t b) {
  const int64_t m = s->m, n = s->n, off = m - 1;
  if ((m + n) * b >= INT32_MAX) raise(SFG_ERR_INVALID_OPERATION, "BDIA: (m + n) * b exceeds the int32 range");
  const int64_t nbr = ceil_div(m, b), rb = std::min(b, m);
  auto* key = dalloc_n<int32_t>(ctx, s->nnz);
  auto* sub = dalloc_n<int32_t>(ctx, s->nnz);
  if (s->nnz)
    SFG_LAUNCH(k_bdia_keys, stream_grid(ctx, s->nnz, kBdiaBlock, 4, 8), kBdiaBlock, 0, ctx->stream, s->row, s->idx,
               s->nnz, (int32_t)b, off, key, sub);
  sfg_tensor* sorted = nullptr;
  try {
    sorted = sort_coo(ctx, nbr, (m + n - 1) * b, s->nnz, key, sub, static_cast<const float*>(s->val), false);
  } catch (...) {
    dfree(ctx, key);
    dfree(ctx, sub);
    throw;
  }
  dfree(ctx, key);
  dfree(ctx, sub);
  sfg_tensor* grid = coo_to_csr(ctx, sorted);  // entries per block row
  free_tensor_arrays(sorted);
  delete sorted;
  auto* cnt = dalloc_n<int32_t>(ctx, nbr);
  sfg_tensor* t = new_tensor(ctx, SFG_BDIA, m, n);
  t->br = t->bc = b;
  t->rb = rb;
  t->nbr = nbr;
  t->ptr = dalloc_n<int32_t>(ctx, nbr + 1);
  const int g = stream_grid(ctx, nbr * 32, kBdiaBlock, 1, 8);
  if (nbr) {
    SFG_LAUNCH(k_bdia_nodes<false>, g, kBdiaBlock, 0, ctx->stream, grid->ptr, grid->idx,
               static_cast<const float*>(grid->val), nbr, (int32_t)b, (int32_t)rb, off, cnt, nullptr, nullptr,
               nullptr);
    scan_counts(ctx, cnt, nbr, t->ptr);
  } else {
    SFG_CUDA(cudaMemsetAsync(t->ptr, 0, 4, ctx->stream));
  }
  int32_t nodes = 0;
  read_back(ctx, t->ptr + nbr, 4, &nodes);
  t->k = nodes;
  t->nnz = (int64_t)nodes * rb;  // values
  t->idx = dalloc_n<int32_t>(ctx, nodes);
  t->val = dalloc_n<float>(ctx, t->nnz);
  if (t->nnz) SFG_CUDA(cudaMemsetAsync(t->val, 0, t->nnz * 4, ctx->stream));
  if (nbr && nodes)
    SFG_LAUNCH(k_bdia_nodes<true>, g, kBdiaBlock, 0, ctx->stream, grid->ptr, grid->idx,
               static_cast<const float*>(grid->val), nbr, (int32_t)b, (int32_t)rb, off, nullptr, t->ptr, t->idx,
               static_cast<float*>(t->val));
  dfree(ctx, cnt);
  free_tensor_arrays(grid);
  delete grid;
  return t;
}

namespace {
// BDIA cells holding a nonzero value, as unordered (row, col, val): a warp
// per block row
__global__ void k_bdia_nonzeros(const int32_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                                const float* __restrict__ val, int64_t nbr, int32_t b, int32_t rb, int64_t m,
                                int32_t* __restrict__ orow, int32_t* __restrict__ ocol, float* __restrict__ oval,
                                unsigned long long* __restrict__ count) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t br = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; br < nbr; br += warps) {
    const int64_t c0 = (int64_t)__ldg(ptr + br) * rb, c1 = (int64_t)__ldg(ptr + br + 1) * rb;
    for (int64_t q0 = c0; q0 < c1; q0 += 32) {
      const int64_t q = q0 + lane;
      const float v = q < c1 ? __ldg(val + q) : 0.f;
      const bool nz = v != 0.f;
      const unsigned msk = __ballot_sync(kFull, nz);
      unsigned long long base = 0;
      if (lane == 0 && msk) base = atomicAdd(count, (unsigned long long)__popc(msk));
      base = __shfl_sync(kFull, base, 0);
      if (nz) {
        const int64_t node = q / rb, r = br * b + (q - node * rb);
        const unsigned long long at = base + __popc(msk & ((1u << lane) - 1u));
        orow[at] = (int32_t)r;
        ocol[at] = (int32_t)(r + __ldg(idx + node));
        oval[at] = v;
      }
    }
  }
}
}  // namespace

sfg_tensor* bdia_to_coo(sfg_context* ctx, const sfg_tensor* t) {
  const int64_t cells = t->k * t->rb;
  auto* r = dalloc_n<int32_t>(ctx, cells);
  auto* c = dalloc_n<int32_t>(ctx, cells);
  auto* v = dalloc_n<float>(ctx, cells);
  auto* count = static_cast<unsigned long long*>(scratch(ctx, 64));
  SFG_CUDA(cudaMemsetAsync(count, 0, 8, ctx->stream));
  if (cells)
    SFG_LAUNCH(k_bdia_nonzeros, stream_grid(ctx, t->nbr * 32, kBdiaBlock, 1, 8), kBdiaBlock, 0, ctx->stream, t->ptr,
               t->idx, static_cast<const float*>(t->val), t->nbr, (int32_t)t->br, (int32_t)t->rb, t->m, r, c, v,
               count);
  unsigned long long nz = 0;
  read_back(ctx, count, 8, &nz);
  sfg_tensor* out = nullptr;
  try {
    out = sort_coo(ctx, t->m, t->n, (int64_t)nz, r, c, v, false);
  } catch (...) {
    for (void* q : {(void*)r, (void*)c, (void*)v}) dfree(ctx, q);
    throw;
  }
  for (void* q : {(void*)r, (void*)c, (void*)v}) dfree(ctx, q);
  return out;
}

}  // namespace sfg

// --------------------------------------------------------------- C2SR(k)
// C2SR(k): map (d0%k, d0/k, d1); merge(0,1), trim(2,2), partition(0)
// (formats.hpp:62-66); plan TileSplit(0,k) Swap(0,1) Sort Fill(1) Fill(0)
// Merge(0) Merge(1) Partition(0). The rows interleaved k ways: row r is
// stored at r' = (r % k) * R + r / k (R = ceil(m/k) rows per residue
// class), a CSR over the kk * R interleaved rows (kk = min(k, m)), and one
// partition per residue class holding entries (storage.hpp:220-231):
// [ptr[j R], ptr[(j+1) R]) when non-empty. Device: the rows rekeyed, the
// canonical radix sort, the CSR row-pointer pass; the kk + 1 class bounds
// are gathered and read back for the (host) partition list.
namespace sfg {
namespace {

__global__ void k_c2sr_rows(const int32_t* __restrict__ row, int64_t nnz, int32_t k, int32_t rr,
                            int32_t* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = ld_stream(row + e);
    out[e] = (r % k) * rr + r / k;
  }
}

__global__ void k_c2sr_bounds(const int32_t* __restrict__ ptr, int32_t kk, int32_t rr, int64_t* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j <= kk) out[j] = __ldg(ptr + (int64_t)j * rr);
}

// original coordinates of a C2SR tensor's entries (a warp per stored row)
__global__ void k_c2sr_coords(const int32_t* __restrict__ ptr, int64_t rows, int32_t k, int32_t rr,
                              int32_t* __restrict__ orow) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < rows; q += warps) {
    const int32_t r = (int32_t)((q % rr) * k + q / rr);
    for (int32_t e = __ldg(ptr + q) + lane; e < __ldg(ptr + q + 1); e += 32) orow[e] = r;
  }
}

}  // namespace

void c2sr_partitions(sfg_context* ctx, sfg_tensor* t) {
  const int32_t kk = (int32_t)t->nbr, rr = (int32_t)t->k;
  auto* b = static_cast<int64_t*>(scratch(ctx, (size_t)(kk + 1) * 8));
  SFG_LAUNCH(k_c2sr_bounds, (int)ceil_div(kk + 1, 256), 256, 0, ctx->stream, t->ptr, kk, rr, b);
  std::vector<int64_t> h(kk + 1);
  SFG_CUDA(cudaMemcpyAsync(h.data(), b, (kk + 1) * 8, cudaMemcpyDeviceToHost, ctx->stream));
  SFG_CUDA(cudaStreamSynchronize(ctx->stream));
  t->partitions.clear();
  for (int32_t j = 0; j < kk; ++j)
    if (h[j + 1] > h[j]) {
      t->partitions.push_back(h[j]);
      t->partitions.push_back(h[j + 1]);
    }
}

sfg_tensor* coo_to_c2sr(sfg_context* ctx, const sfg_tensor* s, int64_t k) {
  const int64_t m = s->m, kk = std::min(k, m), rr = ceil_div(m, k);
  if (kk * rr >= INT32_MAX) raise(SFG_ERR_INVALID_OPERATION, "C2SR: the interleaved rows exceed the int32 range");
  auto* key = dalloc_n<int32_t>(ctx, s->nnz);
  if (s->nnz)
    SFG_LAUNCH(k_c2sr_rows, stream_grid(ctx, s->nnz, kBdiaBlock, 4, 8), kBdiaBlock, 0, ctx->stream, s->row, s->nnz,
               (int32_t)k, (int32_t)rr, key);
  sfg_tensor* sorted = nullptr;
  try {
    sorted = sort_coo(ctx, kk * rr, s->n, s->nnz, key, s->idx, static_cast<const float*>(s->val), false);
  } catch (...) {
    dfree(ctx, key);
    throw;
  }
  dfree(ctx, key);
  sfg_tensor* csr = coo_to_csr(ctx, sorted);
  free_tensor_arrays(sorted);
  delete sorted;
  sfg_tensor* t = new_tensor(ctx, SFG_C2SR, s->m, s->n);
  t->br = t->bc = k;
  t->nbr = kk;
  t->k = rr;
  t->nnz = csr->nnz;
  t->has_zeros = s->has_zeros;
  t->ptr = csr->ptr;
  t->idx = csr->idx;
  t->val = csr->val;
  csr->ptr = csr->idx = nullptr;
  csr->val = nullptr;
  free_tensor_arrays(csr);
  delete csr;
  c2sr_partitions(ctx, t);
  return t;
}

sfg_tensor* c2sr_to_coo(sfg_context* ctx, const sfg_tensor* t) {
  auto* r = dalloc_n<int32_t>(ctx, t->nnz);
  if (t->nnz)
    SFG_LAUNCH(k_c2sr_coords, stream_grid(ctx, t->nbr * t->k, kBdiaBlock / 32, 1, 16), kBdiaBlock, 0, ctx->stream,
               t->ptr, t->nbr * t->k, (int32_t)t->br, (int32_t)t->k, r);
  sfg_tensor* out = nullptr;
  try {
    out = sort_coo(ctx, t->m, t->n, t->nnz, r, t->idx, static_cast<const float*>(t->val), false);
  } catch (...) {
    dfree(ctx, r);
    throw;
  }
  dfree(ctx, r);
  return out;
}

}  // namespace sfg
