// convert_cisr.cu — COO -> CISR(k) and CISR-plus(k) (formats.hpp:67-72).
//
// Reference: map (d0, d1) -> (indirect(d0), d0, d1); merge(0,1), trim(1,2),
// partition(0), with the indirect level computed by the query chain
//   count:    sum(value) groupBy (d0) with value ne 0 -> 1 | otherwise -> 0
//   [plus:    reorder(d0) traverseBy (d0, d1) -> (d0)]
//   schedule: schedule(d0) traverseBy (d0, d1) -> (d0/k) partitions=k
// (query_engine.hpp:202-273). The schedule visits every row of [0, m) —
// the group domain of a bare dimension is dense, so rows without entries
// take part with weight 0 — in ascending row order (CISR: the traverse key
// d0/k, ties by row) or heaviest first, ties by row (CISR-plus: the reorder
// ranks, weight_order), and puts each row on the least-loaded partition
// (the lowest index among equal loads), adding its nonzero count to that
// load. Materialized (storage.hpp:97-234, plan Sum Schedule Sort Merge(0)
// Merge(1) Partition(0)): L0 idx = the partitions holding entries (bounds
// [0, k-1]), L1 ptr + idx = their rows ascending (rows with stored entries,
// explicit zeros included), L2 ptr + idx = each row's columns, values in
// (partition, row, column) order, and one (begin, end) value range per L0
// node (Partition(0), operators.hpp:431-445).
//
// Device plan: the CSR of the input gives each row's entries; a kernel
// counts each row's nonzero values; the greedy schedule — a sequential
// scan over the rows, k loads — runs on the host over the downloaded counts
// (a counting sort by weight gives CISR-plus's visit order); the rows with
// entries are keyed (partition, row) and ordered by the canonical radix
// sort; the L1 / L2 pointers come from scans of the row lengths in that
// order, and a warp per row moves the row's entries.
#include <algorithm>
#include <queue>
#include <vector>

#include "devutil.cuh"
#include "internal.cuh"

namespace sfg {

namespace {

constexpr int kBlock = 256;

void drop(sfg_tensor* t) {  // arrays and the struct
  if (!t) return;
  free_tensor_arrays(t);
  delete t;
}

// nonzero values per row (the count query), and the flag of rows with
// stored entries
__global__ void k_cisr_weights(const int32_t* __restrict__ ptr, const float* __restrict__ val, int64_t m,
                               bool zeros, int32_t* __restrict__ w, int32_t* __restrict__ has) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < m; r += warps) {
    const int32_t s = __ldg(ptr + r), e = __ldg(ptr + r + 1);
    int32_t z = 0;
    if (zeros)
      for (int32_t q = s + lane; q < e; q += 32) z += __ldg(val + q) == 0.f ? 1 : 0;
    z = warp_sum(z);
    if (lane == 0) {
      w[r] = e - s - z;
      has[r] = e > s ? 1 : 0;
    }
  }
}

// rows with entries, keyed (partition, row), in row order
__global__ void k_cisr_keys(const int32_t* __restrict__ has, const int32_t* __restrict__ base,
                            const int32_t* __restrict__ part, int64_t m, int32_t* __restrict__ key,
                            int32_t* __restrict__ sub) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < m; r += (int64_t)gridDim.x * blockDim.x)
    if (__ldg(has + r)) {
      const int32_t q = __ldg(base + r);
      key[q] = __ldg(part + r);
      sub[q] = (int32_t)r;
    }
}

// per L1 node (partition, row): the row's length, and a head flag per
// partition change
__global__ void k_cisr_lengths(const int32_t* __restrict__ skey, const int32_t* __restrict__ srow,
                               const int32_t* __restrict__ ptr, int64_t nr, int32_t* __restrict__ len,
                               int32_t* __restrict__ head) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nr; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = __ldg(srow + i);
    len[i] = __ldg(ptr + r + 1) - __ldg(ptr + r);
    head[i] = (i == 0 || __ldg(skey + i) != __ldg(skey + i - 1)) ? 1 : 0;
  }
}

// L0 idx (partition ids) and L1 ptr over them (the head positions)
__global__ void k_cisr_heads(const int32_t* __restrict__ skey, const int32_t* __restrict__ head,
                             const int32_t* __restrict__ hbase, int64_t nr, int32_t* __restrict__ parts,
                             int32_t* __restrict__ ptr1) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nr; i += (int64_t)gridDim.x * blockDim.x) {
    if (__ldg(head + i)) {
      const int32_t q = __ldg(hbase + i);
      parts[q] = __ldg(skey + i);
      ptr1[q] = (int32_t)i;
    }
    if (i == nr - 1) ptr1[__ldg(hbase + nr)] = (int32_t)nr;
  }
}

// a warp per L1 node moves its row's entries to their new place
__global__ void k_cisr_move(const int32_t* __restrict__ srow, const int32_t* __restrict__ iptr,
                            const int32_t* __restrict__ optr, const int32_t* __restrict__ icol,
                            const float* __restrict__ ival, int64_t nr, int32_t* __restrict__ ocol,
                            float* __restrict__ oval) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < nr; i += warps) {
    const int32_t r = __ldg(srow + i), s = __ldg(iptr + r), e = __ldg(iptr + r + 1), o = __ldg(optr + i);
    for (int32_t q = s + lane; q < e; q += 32) {
      ocol[o + q - s] = __ldg(icol + q);
      oval[o + q - s] = __ldg(ival + q);
    }
  }
}

// CISR -> entries (row, col, val) in (partition, row) order
__global__ void k_cisr_rows(const int32_t* __restrict__ rows, const int32_t* __restrict__ ptr, int64_t nr,
                            int32_t* __restrict__ orow) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < nr; i += warps) {
    const int32_t r = __ldg(rows + i);
    for (int32_t q = __ldg(ptr + i) + lane; q < __ldg(ptr + i + 1); q += 32) orow[q] = r;
  }
}

// The schedule query on the host: rows visited in order (or heaviest first
// for CISR-plus, ties by row), each to the least-loaded partition, the
// lowest index among equal loads (query_engine.hpp:220-262).
std::vector<int32_t> schedule_rows(const std::vector<int32_t>& w, int64_t k, bool plus) {
  const int64_t m = (int64_t)w.size();
  std::vector<int32_t> part(m);
  using Load = std::pair<int64_t, int64_t>;  // (load, partition)
  std::priority_queue<Load, std::vector<Load>, std::greater<Load>> heap;
  for (int64_t p = 0; p < k; ++p) heap.push({0, p});
  auto place = [&](int64_t r) {
    Load top = heap.top();
    heap.pop();
    part[r] = (int32_t)top.second;
    top.first += w[r];
    heap.push(top);
  };
  if (!plus) {
    for (int64_t r = 0; r < m; ++r) place(r);
  } else {
    // counting sort by weight, descending; rows ascending within a weight
    int32_t wmax = 0;
    for (int32_t x : w) wmax = std::max(wmax, x);
    std::vector<int64_t> start(wmax + 2, 0);
    for (int32_t x : w) ++start[wmax - x + 1];
    for (int32_t b = 1; b <= wmax + 1; ++b) start[b] += start[b - 1];
    std::vector<int64_t> order(m);
    for (int64_t r = 0; r < m; ++r) order[start[wmax - w[r]]++] = r;
    for (int64_t r : order) place(r);
  }
  return part;
}

}  // namespace

sfg_tensor* coo_to_cisr(sfg_context* ctx, const sfg_tensor* s, int64_t k, bool plus) {
  const int64_t m = s->m;
  if (k <= 0) raise(SFG_ERR_INVALID_OPERATION, "CISR: the partition count must be positive");
  sfg_tensor* csr = coo_to_csr(ctx, s);
  int32_t *w = nullptr, *has = nullptr, *base = nullptr, *part = nullptr;
  auto release = [&] {
    for (void* q : {(void*)w, (void*)has, (void*)base, (void*)part}) dfree(ctx, q);
    drop(csr);
  };
  sfg_tensor* t = new_tensor(ctx, plus ? SFG_CISRP : SFG_CISR, m, s->n);
  try {
    w = dalloc_n<int32_t>(ctx, m);
    has = dalloc_n<int32_t>(ctx, m);
    base = dalloc_n<int32_t>(ctx, m + 1);
    SFG_LAUNCH(k_cisr_weights, stream_grid(ctx, m, kBlock / 32, 1, 16), kBlock, 0, ctx->stream, csr->ptr,
               static_cast<const float*>(csr->val), m, s->has_zeros != 0, w, has);
    scan_counts(ctx, has, m, base);
    // the schedule over the downloaded row weights
    std::vector<int32_t> hw(m);
    int32_t nr = 0;
    SFG_CUDA(cudaMemcpyAsync(hw.data(), w, m * 4, cudaMemcpyDeviceToHost, ctx->stream));
    read_back(ctx, base + m, sizeof nr, &nr);
    const std::vector<int32_t> hpart = schedule_rows(hw, k, plus);
    part = dalloc_n<int32_t>(ctx, m);
    SFG_CUDA(cudaMemcpyAsync(part, hpart.data(), m * 4, cudaMemcpyHostToDevice, ctx->stream));
    // rows with entries ordered by (partition, row)
    int32_t* key = dalloc_n<int32_t>(ctx, nr);
    int32_t* sub = dalloc_n<int32_t>(ctx, nr);
    SFG_LAUNCH(k_cisr_keys, stream_grid(ctx, m, kBlock, 4, 8), kBlock, 0, ctx->stream, has, base, part, m, key, sub);
    sfg_tensor* srt = nullptr;
    try {
      srt = sort_coo(ctx, k, m, nr, key, sub, reinterpret_cast<const float*>(sub), false);  // payload unused
    } catch (...) {
      dfree(ctx, key);
      dfree(ctx, sub);
      throw;
    }
    dfree(ctx, key);
    dfree(ctx, sub);
    // L1 / L2 pointers, L0 nodes
    int32_t* len = dalloc_n<int32_t>(ctx, nr);
    int32_t* head = dalloc_n<int32_t>(ctx, nr);
    int32_t* hbase = dalloc_n<int32_t>(ctx, nr + 1);
    t->ptr = dalloc_n<int32_t>(ctx, nr + 1);
    if (nr) {
      SFG_LAUNCH(k_cisr_lengths, stream_grid(ctx, nr, kBlock, 4, 8), kBlock, 0, ctx->stream, srt->row, srt->idx,
                 csr->ptr, nr, len, head);
      scan_counts(ctx, len, nr, t->ptr);
      scan_counts(ctx, head, nr, hbase);
    } else {
      SFG_CUDA(cudaMemsetAsync(t->ptr, 0, 4, ctx->stream));
    }
    int32_t np = 0;
    if (nr) read_back(ctx, hbase + nr, sizeof np, &np);
    t->k = np;
    t->slots = dalloc_n<int32_t>(ctx, np);
    t->ptr1 = dalloc_n<int32_t>(ctx, np + 1);
    if (nr)
      SFG_LAUNCH(k_cisr_heads, stream_grid(ctx, nr, kBlock, 4, 8), kBlock, 0, ctx->stream, srt->row, head, hbase,
                 nr, t->slots, t->ptr1);
    else
      SFG_CUDA(cudaMemsetAsync(t->ptr1, 0, 4, ctx->stream));
    t->nnr = nr;
    t->row = srt->idx;  // L1 idx: the rows, partition by partition
    srt->idx = nullptr;
    t->nnz = csr->nnz;
    t->idx = dalloc_n<int32_t>(ctx, t->nnz);
    t->val = dalloc_n<float>(ctx, t->nnz);
    if (nr)
      SFG_LAUNCH(k_cisr_move, stream_grid(ctx, nr, kBlock / 32, 1, 16), kBlock, 0, ctx->stream, t->row, csr->ptr,
                 t->ptr, csr->idx, static_cast<const float*>(csr->val), nr, t->idx, static_cast<float*>(t->val));
    t->br = t->bc = k;
    t->has_zeros = s->has_zeros;
    // Partition(0): the value range of each present partition
    std::vector<int32_t> p1(np + 1), p2(nr + 1);
    SFG_CUDA(cudaMemcpyAsync(p1.data(), t->ptr1, (np + 1) * 4, cudaMemcpyDeviceToHost, ctx->stream));
    SFG_CUDA(cudaMemcpyAsync(p2.data(), t->ptr, (nr + 1) * 4, cudaMemcpyDeviceToHost, ctx->stream));
    SFG_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int32_t q = 0; q < np; ++q) {
      t->partitions.push_back(p2[p1[q]]);
      t->partitions.push_back(p2[p1[q + 1]]);
    }
    for (void* q : {(void*)len, (void*)head, (void*)hbase}) dfree(ctx, q);
    drop(srt);
  } catch (...) {
    drop(t);
    release();
    throw;
  }
  release();
  return t;
}

sfg_tensor* cisr_to_coo(sfg_context* ctx, const sfg_tensor* t) {
  auto* r = dalloc_n<int32_t>(ctx, t->nnz);
  if (t->nnr)
    SFG_LAUNCH(k_cisr_rows, stream_grid(ctx, t->nnr, kBlock / 32, 1, 16), kBlock, 0, ctx->stream, t->row, t->ptr,
               t->nnr, r);
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
