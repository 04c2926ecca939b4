// internal.cuh — shared host/device plumbing for the sm_100a sparse path.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <map>
#include <unordered_map>
#include <vector>
#include <cstdint>
#include <string>

#include "../../include/sparseforge_b200.h"

namespace sfg {

// ------------------------------------------------------------------ errors
struct Failure {
  int code;
  std::string msg;
};

[[noreturn]] void raise(int code, const std::string& msg);
[[noreturn]] void raise_cuda(cudaError_t e, const char* what, const char* file, int line);
void set_last_error(const std::string& msg);

#define SFG_CUDA(call)                                                      \
  do {                                                                      \
    cudaError_t e__ = (call);                                               \
    if (e__ != cudaSuccess) ::sfg::raise_cuda(e__, #call, __FILE__, __LINE__); \
  } while (0)

extern std::atomic<int64_t> g_launches;
bool debug_launches();  // SFG_DEBUG=1: trace and synchronize every launch
void trace_launch(const char* name, cudaStream_t stream);

// Every kernel launch goes through here: counted (bench gpu_launches) and
// checked for launch-configuration errors.
#define SFG_LAUNCH(kernel, grid, block, smem, stream, ...)                   \
  do {                                                                      \
    if (::sfg::debug_launches()) ::sfg::trace_launch(#kernel, (stream));    \
    kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);             \
    ::sfg::g_launches.fetch_add(1, std::memory_order_relaxed);              \
    SFG_CUDA(cudaPeekAtLastError());                                        \
    if (::sfg::debug_launches()) SFG_CUDA(cudaStreamSynchronize(stream));   \
  } while (0)

}  // namespace sfg

// ---------------------------------------------------------------- context
struct sfg_context {
  int device = 0;
  cudaStream_t stream = nullptr;
  int sms = 148;
  size_t total_mem = 0;         // device memory (bytes)
  int64_t* pinned = nullptr;   // small host scratch for size read-backs
  cudaEvent_t sizes_ev = nullptr;  // read_back_async completion
  // Deferred size read-backs owned by tensors (core.cu: size slots): pinned
  // words, one completion event each, and the free list.
  int32_t* size_slots = nullptr;
  std::vector<cudaEvent_t> size_events;
  std::vector<int> free_size_slots;
  char* staging = nullptr;     // pinned host staging for file ingest (grow-only)
  size_t staging_bytes = 0;
  void* scratch = nullptr;     // device scratch (counters, histograms, flags)
  size_t scratch_bytes = 0;
  void* status = nullptr;      // look-back status words only
  size_t status_words = 0;
  uint32_t epoch = 1;          // look-back status generation
  // Block cache over the stream-ordered pool (core.cu: dalloc/dfree). All
  // work of a context runs on ctx->stream, so a freed block can be handed
  // out again at once: stream order serialises its old and new users.
  std::multimap<size_t, void*> free_blocks;     // size class -> block
  std::unordered_map<void*, size_t> block_size;  // every cached-or-live block
  size_t cached_bytes = 0;
};

// ------------------------------------------------------------------ tensor
// Device-resident materialized tensor. Array roles per format (the level
// arrays of MaterializedTensor, storage.hpp:77-91):
//   COO : row[nnz] (L0 idx), idx[nnz] (L1 idx)
//   CSR : ptr[m+1], idx[nnz]              CSC: ptr[n+1], idx[nnz] (rows)
//   DCSR: row[nnr] (L0 idx), ptr[nnr+1], idx[nnz]
//   DCSC: row[nnr] = the nonempty columns (L0 idx), ptr[nnr+1], idx[nnz] = rows
//   DIAV: slots[K] (diagonals), val[K*n] (dense vector over the columns)
//   CISR: slots[K] (present partitions, L0 idx), ptr1[K+1] + row[nnr] (L1:
//         rows per partition), ptr[nnr+1] + idx[nnz] (L2), val[nnz]
//   ELL : slots[K] (L0 idx), idx[K*m] (L2 idx, slot-major), val[K*m]
//   BCSR: ptr[nbr+1], idx[nblocks] (bcol), val[nblocks*rb*cb] block-major
//   HYB : part[0] = ELL of the remainder, part[1] = COO of the selection
//   HBELL: part[0] = BELL(b) of the dense blocks, part[1] = COO of the rest
//   BELL: slots[K], idx[K*nbr] (block column of cell (slot, block row),
//         slot-major), val[K*nbr*rb*cb]; nnz = K*nbr cells
//   DOK : val = records {row, col, val}[nnz];  LIL: ptr[m+1], val = {col, val}[nnz]
//   DIA : slots[K] (diagonals col - row, ascending), val[K*m]; nnz = K*m
//   BDIA: ptr[nbr+1], idx[K] (diagonals per block row), val[K*rb]; k = K, nnz = K*rb
//   C2SR: ptr[kk*R+1] over the interleaved rows (row' = (r % k) * R + r / k,
//         R = ceil(m/k), kk = min(k, m); nbr = kk, k = R), idx, val; partitions
//   CSB : ptr[nbr*nbc+1] over the block grid, row[nnz] (row in block),
//         idx[nnz] (column in block), val[nnz]
struct sfg_tensor {
  sfg_context* ctx = nullptr;
  int32_t kind = SFG_COO;
  int32_t dtype = SFG_F32;
  int64_t m = 0, n = 0;
  int64_t nnz = 0;       // stored coordinates (COO/CSR/CSC/DCSR), cells (ELL), blocks (BCSR)
  int64_t nnr = 0;       // DCSR nonempty rows (read via tensor_nnr: may still be in flight)
  int32_t nnr_slot = -1; // >= 0: nnr is being read back into this size slot
  int64_t k = 0;         // ELL slots
  int64_t br = 0, bc = 0;        // BCSR block shape (r, c)
  int64_t rb = 0, cb = 0;        // BCSR level-2/3 extents (== r, c except one-tile edge)
  int64_t nbr = 0, nbc = 0;      // BCSR block grid
  int64_t threshold = 0;         // HYB min_sum
  int32_t has_zeros = -1;        // COO: explicit zero values present? 1/0, -1 unknown
  uint32_t* tc_plan = nullptr;   // BCSR: cached tensor-core SpMM plan (bcsr_tc.cu)
  int32_t* tc_base = nullptr;    //   and its stage schedule: per-group first stage,
  uint32_t* tc_desc = nullptr;   //   stage descriptors
  int32_t* row = nullptr;
  int32_t* ptr = nullptr;
  int32_t* idx = nullptr;
  int32_t* slots = nullptr;
  int32_t* ptr1 = nullptr;  // CISR: L1 ptr over the present partitions
  void* val = nullptr;
  sfg_tensor* part[2] = {nullptr, nullptr};
  std::vector<int64_t> partitions;  // C2SR / CISR: (begin, end) value ranges, host
};

namespace sfg {

// Stream-ordered device allocation through the context's block cache (a
// conversion allocates the same large arrays every call; growing the
// driver pool for them costs milliseconds of host time per call).
void* dalloc(sfg_context* ctx, size_t bytes);
void dfree(sfg_context* ctx, void* p);
// Returns every cached (free) block to the pool.
void release_cached(sfg_context* ctx);
template <class T>
T* dalloc_n(sfg_context* ctx, int64_t n) {
  return static_cast<T*>(dalloc(ctx, static_cast<size_t>(n > 0 ? n : 1) * sizeof(T)));
}

// Adds carry slots (row[i] >= 0: partial sum val[i * nd ...] of that row;
// runs of equal rows are consecutive) to C in slot order, without atomics:
// a log-32 tree of k_carry_level passes (spmm.cu). Deterministic.
void carry_fix(sfg_context* ctx, const int32_t* row, const float* val, int64_t n, int nd, float* c, int64_t ldc);

// Scratch with at least `bytes` bytes (grows; contents undefined). Never
// used for look-back status words.
void* scratch(sfg_context* ctx, size_t bytes);
// Dedicated look-back status words (>= `words`), zero-filled whenever the
// buffer is (re)allocated and written only by look-back kernels, so a stale
// word always carries an older epoch than the launch reading it.
unsigned long long* lookback_status(sfg_context* ctx, size_t words);
// Copy `count` int64 values device->host through pinned memory and sync.
void read_back(sfg_context* ctx, const void* dev, size_t bytes, void* host);
// The same in two halves, so the host can enqueue more work before it
// waits: start copies `bytes` (<= 1 KB) at this point of the stream, wait
// blocks until they arrived. One outstanding read at a time per context.
void read_back_start(sfg_context* ctx, const void* dev, size_t bytes);
// Deferred 4-byte read-back into a size slot (-1: none free, read now).
int size_slot_start(sfg_context* ctx, const int32_t* dev);
int32_t size_slot_finish(sfg_context* ctx, int slot);
// A DCSR's nonempty-row count, waiting for its read-back if still pending.
int64_t tensor_nnr(const sfg_tensor* t);
void read_back_wait(sfg_context* ctx, size_t bytes, void* host);

sfg_tensor* new_tensor(sfg_context* ctx, int kind, int64_t m, int64_t n);
void free_tensor_arrays(sfg_tensor* t);

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Grid for a grid-stride streaming kernel: a few waves of resident CTAs.
inline int stream_grid(const sfg_context* ctx, int64_t work_items, int block, int per_thread,
                       int ctas_per_sm = 8) {
  int64_t want = ceil_div(work_items, static_cast<int64_t>(block) * per_thread);
  int64_t cap = static_cast<int64_t>(ctx->sms) * ctas_per_sm;
  if (want < 1) want = 1;
  return static_cast<int>(want < cap ? want : cap);
}

// ----------------------------------------------------- kernel entry points
// (defined in the per-area .cu files, called from abi.cu)
// Validates a caller-sorted COO; returns 1 when it holds explicit zero values.
int check_coo_canonical(sfg_context* ctx, const int32_t* row, const int32_t* col, const float* val, int64_t m,
                         int64_t n, int64_t nnz);
// Whole file -> the context's pinned staging by parallel reads (and, with
// `dev`, a device copy); returns the host bytes (NUL-terminated).
char* read_file_pinned(sfg_context* ctx, const char* path, int64_t* size, char** dev);
// USPT container (container.cu, io.hpp:202-334).
void write_container(sfg_context* ctx, const sfg_tensor* t, const char* path);
sfg_tensor* read_container(sfg_context* ctx, const char* path, const sfg_format* fmt /* null: infer */);
// Dense C = A B over two sparse operands (spgemm.cu).
void spgemm(sfg_context* ctx, const sfg_tensor* a, const sfg_tensor* b, float* c, int64_t ldc, bool accumulate);
// Matrix Market file -> canonical COO (mm_read.cu).
sfg_tensor* read_matrix_market(sfg_context* ctx, const char* path, bool sum_duplicates);
sfg_tensor* sort_coo(sfg_context* ctx, int64_t m, int64_t n, int64_t nnz, const int32_t* row,
                     const int32_t* col, const float* val, bool sum_duplicates);
// `hist`: the digit histograms of the keys (8 bits per pass, 256 counts per
// pass, in the context scratch buffer), when the caller built them while
// writing the keys; null = computed here.
// rowpart.cu (row-partitioned multi-GPU path)
void comm_unique_id(uint8_t* out);
sfg_comm* comm_create(sfg_context* ctx, int32_t nranks, int32_t rank, const uint8_t* id);
void comm_destroy(sfg_comm* c);
void allgather_chunks(sfg_context* ctx, sfg_comm* c, float* buf, int64_t chunk_elems);
void rowpart_spmv(sfg_context* ctx, sfg_comm* c, const sfg_tensor* a, const float* x, float* y, int64_t chunk_rows,
                  bool gather);
void rowpart_spmm(sfg_context* ctx, sfg_comm* c, const sfg_tensor* a, const void* b, int b_dtype, int64_t nd,
                  int64_t ldb, float* cbuf, int64_t chunk_rows, bool gather);

void radix_sort(sfg_context* ctx, uint64_t* keys, uint32_t* pay, int64_t n, int key_bits,
                uint64_t** kres, uint32_t** pres, uint64_t** kalt, uint32_t** palt,
                uint32_t* hist = nullptr);
// ptr[extent+1] + copies of (other, val) from entries sorted by `key`.
void compress_sorted(sfg_context* ctx, const int32_t* key, const int32_t* other, const float* val,
                     int64_t nnz, int64_t extent, int32_t* ptr, int32_t* oidx, float* oval);
void sort_u64_keys(sfg_context* ctx, uint64_t* keys, int64_t n, int key_bits, uint64_t** sorted_out);

sfg_tensor* coo_to_coo(sfg_context* ctx, const sfg_tensor* s);
// Non-COO sources (convert_src.cu): dematerialize, then the COO paths.
sfg_tensor* convert_from_compressed(sfg_context* ctx, const sfg_tensor* s, const sfg_format& dst);
sfg_tensor* coo_to_csr(sfg_context* ctx, const sfg_tensor* s);
sfg_tensor* coo_to_csc(sfg_context* ctx, const sfg_tensor* s);
sfg_tensor* coo_to_dcsr(sfg_context* ctx, const sfg_tensor* s);
sfg_tensor* coo_to_ell(sfg_context* ctx, const sfg_tensor* s);
sfg_tensor* coo_to_bcsr(sfg_context* ctx, const sfg_tensor* s, int64_t r, int64_t c, int dtype);
// per-entry flags of the block-count rule over canonical COO (false: grid too
// wide for the shared counters — the caller sorts instead)
bool block_nz_flags(sfg_context* ctx, const sfg_tensor* s, int64_t r, int64_t c, int64_t min_sum, uint8_t* flag);
sfg_tensor* coo_to_hyb(sfg_context* ctx, const sfg_tensor* s, int64_t min_sum);
// DIA and CSB(r,c) (convert_dia.cu), and back to canonical COO (DIA: its
// nonzero cells; CSB: every entry).
sfg_tensor* coo_to_dia(sfg_context* ctx, const sfg_tensor* s, bool variant = false);  // variant: DIA-variant
sfg_tensor* coo_to_csb(sfg_context* ctx, const sfg_tensor* s, int64_t br, int64_t bc);
sfg_tensor* dia_to_coo(sfg_context* ctx, const sfg_tensor* t);  // DIA or DIA-variant
sfg_tensor* coo_to_dcsc(sfg_context* ctx, const sfg_tensor* s);
sfg_tensor* coo_to_cisr(sfg_context* ctx, const sfg_tensor* s, int64_t k, bool plus);
sfg_tensor* cisr_to_coo(sfg_context* ctx, const sfg_tensor* t);
sfg_tensor* dcsc_to_coo(sfg_context* ctx, const sfg_tensor* t);
sfg_tensor* csb_to_coo(sfg_context* ctx, const sfg_tensor* t);
sfg_tensor* coo_to_bdia(sfg_context* ctx, const sfg_tensor* s, int64_t b);
sfg_tensor* bdia_to_coo(sfg_context* ctx, const sfg_tensor* t);  // nonzero cells
sfg_tensor* coo_to_c2sr(sfg_context* ctx, const sfg_tensor* s, int64_t k);
sfg_tensor* c2sr_to_coo(sfg_context* ctx, const sfg_tensor* t);
// C2SR partitions from its row pointers (R rows per residue class).
void c2sr_partitions(sfg_context* ctx, sfg_tensor* t);
// Exclusive scan of n int32 counts into ptr[0..n] (convert_bcsr.cu).
void scan_counts(sfg_context* ctx, const int32_t* cnt, int64_t n, int32_t* ptr);
// The nonzero entries of an ELL / BELL tensor as a canonical COO (convert_src.cu).
sfg_tensor* ell_nonzeros_to_coo(sfg_context* ctx, const sfg_tensor* s);
// Blocked ELL (convert_bell.cu): the BCSR blocks relaid slot by slot.
sfg_tensor* coo_to_bell(sfg_context* ctx, const sfg_tensor* s, int64_t b);
// decompose by blocks (the block count rule) and the hybrid BELL/COO built on
// it: part[0] = BELL(b) of the blocks with >= min_sum nonzeros, part[1] = COO.
void decompose_blocks(sfg_context* ctx, const sfg_tensor* s, int64_t r, int64_t c, int64_t min_sum,
                      sfg_tensor** sel, sfg_tensor** rem);
sfg_tensor* coo_to_hbell(sfg_context* ctx, const sfg_tensor* s, int64_t b, int64_t min_sum);
// Value-layout formats (pack.cu): Pack(0,1) over COO (DOK) / CSR (LIL).
sfg_tensor* coo_to_dok(sfg_context* ctx, const sfg_tensor* s);
sfg_tensor* coo_to_lil(sfg_context* ctx, const sfg_tensor* s);
// A DOK / LIL tensor as separate arrays (new device arrays; row only for
// DOK), e.g. for the container writer. The caller frees them (dfree).
void aos_unpack(sfg_context* ctx, const sfg_tensor* t, int32_t** row, int32_t** idx, float** val);
// A DOK / LIL tensor as a new COO / CSR tensor (the same entries, SoA).
sfg_tensor* aos_to_soa(sfg_context* ctx, const sfg_tensor* t);
// The reverse: records from separate arrays (t->val must hold nnz records).
void aos_pack_into(sfg_context* ctx, sfg_tensor* t, const int32_t* row, const int32_t* idx, const float* val);
void decompose_rows(sfg_context* ctx, const sfg_tensor* s, int64_t min_sum, sfg_tensor** sel,
                    sfg_tensor** rem, int32_t* totals);
void row_partition(sfg_context* ctx, const sfg_tensor* coo, int parts, int64_t* bounds);
// The same rule over a host row array (no device work).
void row_bounds_host(const int32_t* rows, int64_t nnz, int64_t m, int parts, int64_t* bounds);
sfg_tensor* coo_slice_rows(sfg_context* ctx, const sfg_tensor* coo, int64_t r0, int64_t r1);

void spmv(sfg_context* ctx, const sfg_tensor* a, const float* x, float* y, bool accumulate);
void spmm(sfg_context* ctx, const sfg_tensor* a, const void* b, int b_dtype, int64_t nd,
          int64_t ldb, float* c, int64_t ldc, bool accumulate);

sfg_tensor* gen_uniform(sfg_context* ctx, uint64_t seed, int64_t m, int64_t n, int per_row);
sfg_tensor* gen_from_keys(sfg_context* ctx, uint64_t seed, int kind, int scale, int64_t m,
                          int64_t n, int64_t draws);
void gen_dense(sfg_context* ctx, uint64_t seed, int64_t count, float* out);
sfg_tensor* gen_block_sparse(sfg_context* ctx, uint64_t seed, int64_t m, int64_t n, int64_t r,
                             int64_t c, uint32_t thresh, int dtype);

}  // namespace sfg
