/* sparseforge_b200.h — C-ABI of the B200-native sparse hot path.
 *
 * Drop-in boundary for the reference's hot path (sparse-forge,
 * /root/reference/proj/include/sparseforge): COO ingest, conversion to
 * CSR/CSC/DCSR/ELL/BCSR/hybrid ELL+COO, decompose, and SpMV/SpMM. Plain
 * pointers and sizes, no C++ or torch types. Every entry point names the
 * reference interface it replaces (file:line relative to proj/include/).
 *
 * Data model. Tensors live in device memory, owned by opaque sfg_tensor
 * handles. Indices are int32, values fp32 (bf16 optional for BCSR); the
 * reference uses int64 / f64. Conversions are permutations and paddings, so
 * arrays widened to int64 / f64 equal the reference's MaterializedTensor
 * (storage.hpp:77-91) bit for bit. Kernels accumulate in fp32.
 *
 * Execution model. Every call is ordered on the context's CUDA stream.
 * Calls whose output sizes are data dependent (from_coo, DCSR, ELL,
 * BCSR, decompose) read those sizes back with one small synchronous copy.
 * A context or a tensor is not thread-safe; several contexts on several
 * streams are.
 *
 * Errors. Status 0 is success; 1 + ErrorKind (errors.hpp:10-21) for the
 * reference's semantic errors; SFG_ERR_CUDA / SFG_ERR_OOM for device
 * failures. sfg_last_error() returns a thread-local message. There is no
 * CPU fallback: without a usable sm_100a device every compute call fails
 * with SFG_ERR_CUDA.
 */
#ifndef SPARSEFORGE_B200_H
#define SPARSEFORGE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ----------------------------------------------------------------- status */
enum sfg_status {
  SFG_OK = 0,
  /* 1 + sparseforge::ErrorKind (errors.hpp:10-21) */
  SFG_ERR_PARSE = 1,
  SFG_ERR_NON_AFFINE = 2,
  SFG_ERR_NON_INTEGRAL = 3,
  SFG_ERR_UNSUPPORTED_SOURCE = 4,
  SFG_ERR_UNSUPPORTED_HEADER = 5,
  SFG_ERR_DUPLICATE_COORDINATE = 6,
  SFG_ERR_COLLISION = 7,
  SFG_ERR_INVALID_OPERATION = 8,
  SFG_ERR_SINGULAR = 9,
  SFG_ERR_IO = 10,
  /* device-side failures (no reference equivalent) */
  SFG_ERR_CUDA = 64,
  SFG_ERR_OOM = 65,
  SFG_ERR_NCCL = 66,
};

/* ---------------------------------------------------------------- formats */
/* The named formats of formats.hpp:32-88 that the hot path covers, plus the
 * hybrid ELL+COO pair produced by decompose (decompose.hpp:30). */
enum sfg_format_kind {
  SFG_COO = 0,  /* map (d0,d1)->(d0,d1); trim(0,1)               formats.hpp:39 */
  SFG_CSR = 1,  /* map (d0,d1)->(d0,d1); merge(0), trim(1,1)     formats.hpp:41 */
  SFG_CSC = 2,  /* map (d0,d1)->(d1,d0); merge(0), trim(1,1)     formats.hpp:42 */
  SFG_DCSR = 3, /* map (d0,d1)->(d0,d1); merge(0), trim(0,1)     formats.hpp:43 */
  SFG_ELL = 4,  /* (indirect(d1), d0, d1) + sum/enum chain      formats.hpp:59-61 */
  SFG_BCSR = 5, /* (d0/r, d1/c, d0%r, d1%c); merge(0), trim(1,1) formats.hpp:49-53 */
  SFG_HYB = 6,  /* decompose by row count >= threshold: selected rows -> COO,
                   remaining rows -> ELL (the hybrid ELL+COO format)          */
  /* Value-layout formats: Pack(0,1) (operators.hpp:424-430) stores the
   * level-0..1 coordinates and the value of each entry as one record (AoS,
   * storage.hpp:128-133) instead of separate arrays (SoA).                 */
  SFG_DOK = 7,  /* COO + pack(0,1): records {row, col, val}      formats.hpp:40 */
  SFG_LIL = 8,  /* CSR + pack(0,1): ptr[m+1] + records {col, val} formats.hpp:45 */
  SFG_BELL = 9, /* blocked ELL: (indirect(d1/b), d0/b, d1/b, d0%b, d1%b) + block
                   count / slot chain, slot-major b x b blocks  formats.hpp:79-85 */
  SFG_DIA = 10, /* map (d0,d1)->(d1-d0, d0); merge(0), trim(0,0) formats.hpp:46 */
  SFG_CSB = 11, /* (d0/r, d1/c, d0%r, d1%c); merge(0,1), trim(2,3) formats.hpp:54-57 */
  SFG_BDIA = 12, /* (d0/b, d1-d0, d0%b); merge(0), trim(1,1)     formats.hpp:76-79 */
  SFG_C2SR = 13, /* (d0%k, d0/k, d1); merge(0,1), trim(2,2), partition(0)
                    formats.hpp:62-66 — rows interleaved k ways, entry ranges
                    per residue class as partitions                          */
  SFG_HBELL = 14, /* hybrid BELL/COO (the paper's GPU format, PAPER.md fig.
                     BELL-COO): decompose by b x b blocks with >= threshold
                     nonzeros -> BELL(b), the rest -> COO                    */
  SFG_DCSC = 15, /* (d1, d0); merge(0), trim(0,1): nonempty columns, then
                    rows                                      formats.hpp:43 */
  SFG_DIAV = 16, /* DIA-variant: (d1-d0, d1); merge(0), trim(0,0) — diagonals
                    over a dense vector of columns            formats.hpp:47 */
  SFG_CISR = 17, /* (indirect(d0), d0, d1); merge(0,1), trim(1,2), partition(0)
                    with the row count + greedy schedule onto k partitions
                    (rows in order)                        formats.hpp:67-72 */
  SFG_CISRP = 18, /* CISR-plus: rows visited heaviest first (reorder query) */
};

enum sfg_dtype { SFG_F32 = 0, SFG_BF16 = 1 };

typedef struct sfg_format {
  int32_t kind;        /* sfg_format_kind */
  int32_t block_r;     /* BCSR / CSB block rows (r); BELL / BDIA block size (b); C2SR k */
  int32_t block_c;     /* BCSR / CSB block columns (c); BELL: b         */
  int32_t value_dtype; /* sfg_dtype of stored values (BF16: BCSR only) */
  int64_t threshold;   /* HYB / HBELL: DecomposeRule::min_sum (decompose.hpp:17-20) */
} sfg_format;

/* LevelStorage flags (storage.hpp:17-22). */
enum { SFG_LEVEL_SIZE = 1, SFG_LEVEL_PTR = 2, SFG_LEVEL_IDX = 4, SFG_LEVEL_DENSE_VECTOR = 8 };

typedef struct sfg_context sfg_context;
typedef struct sfg_tensor sfg_tensor;
typedef struct sfg_comm sfg_comm; /* NCCL communicator of the row-partitioned path */

/* One level of a MaterializedTensor (storage.hpp:77-83); device pointers. */
typedef struct sfg_level_view {
  uint32_t storage;   /* SFG_LEVEL_* */
  int64_t lo, hi;     /* Interval bounds */
  int64_t node_count;
  int64_t idx_len, ptr_len;
  const int32_t* idx; /* device */
  const int32_t* ptr; /* device */
} sfg_level_view;

typedef struct sfg_tensor_view {
  int32_t kind;       /* sfg_format_kind */
  int32_t value_dtype;
  int64_t rows, cols; /* logical shape */
  int32_t nlevels;
  sfg_level_view level[5]; /* BELL has five levels */
  int64_t nvals;
  const void* values; /* device */
  const sfg_tensor* parts[2]; /* SFG_HYB: {ELL of remainder, COO of selection} */
  /* ValueLayout (tensor.hpp:58-64): 0 SoA, 1 AoS over levels
   * [aos_start, aos_end] (the Pack span). With AoS, the idx arrays of the
   * packed levels and the values are interleaved records of record_words
   * 32-bit words: element i of such an array is at pointer[i * record_words]. */
  int32_t layout;
  int32_t aos_start, aos_end;
  int32_t record_words; /* 1 for SoA */
  /* Partition(level) (operators.hpp:431-445, storage.hpp:220-231): value
   * ranges [begin, end) per coordinate of the partition level, as
   * npartitions (begin, end) pairs in HOST memory owned by the tensor. */
  int64_t npartitions;
  const int64_t* partitions;
} sfg_tensor_view;

/* --------------------------------------------------------------- context */
const char* sfg_last_error(void);
/* stream: a cudaStream_t, or NULL for the legacy default stream. */
int sfg_context_create(int device, void* stream, sfg_context** out);
/* Waits for the old stream before switching (cached blocks move with it). */
int sfg_context_set_stream(sfg_context* ctx, void* stream);
int sfg_context_destroy(sfg_context* ctx);
int sfg_context_synchronize(sfg_context* ctx);
/* Device memory freed by tensors stays cached in the context for the next
 * conversion; this returns the cached blocks to the driver pool. bytes_out
 * (optional) receives how many bytes were cached before the call. */
int sfg_context_release_cached(sfg_context* ctx, int64_t* bytes_out);

/* ------------------------------------------------------- format / planner */
/* resolve_format (formats.hpp:92-125) for the names above: "COO", "CSR",
 * "CSC", "DCSR", "ELL", "BCSR(r,c)" (BCSR(r) = BCSR(r,r); BCSR = (2,2)) and
 * the hybrid "HYB(T)". Unknown names -> SFG_ERR_PARSE. */
int sfg_format_resolve(const char* text, sfg_format* out);
/* plan_conversion + plan_lines (planner.hpp:95-252, 22-27) for a COO
 * source: the op list the device path executes, one op per line. */
int sfg_plan_text(const sfg_format* src, const sfg_format* dst, char* buf, int64_t len);
/* explain_storage(infer_storage(fmt)) (storage.hpp:35-75). */
int sfg_storage_explain(const sfg_format* fmt, char* buf, int64_t len);

/* ---------------------------------------------------------------- ingest */
enum {
  SFG_FLAG_SORTED = 1,          /* input already (row,col)-sorted and unique */
  SFG_FLAG_SUM_DUPLICATES = 2,  /* from_coo(..., sum_duplicates=true) */
  SFG_FLAG_HOST = 4,            /* pointers are host memory */
};

/* from_coo (tensor.hpp:118-162): range check -> InvalidOperation; stable
 * (row,col) sort (device LSD radix sort); duplicates -> DuplicateCoordinate,
 * or summed in sorted order with SFG_FLAG_SUM_DUPLICATES. Copies the input. */
int sfg_from_coo(sfg_context* ctx, int64_t rows, int64_t cols, int64_t nnz, const int32_t* row,
                 const int32_t* col, const float* val, uint32_t flags, sfg_tensor** out);

/* ------------------------------------------------------------- conversion */
/* convert_structure(COO -> dst) + materialize(infer_storage(dst))
 * (planner.hpp:261-265, 254-257; storage.hpp:97-234). src must be COO. */
int sfg_convert(sfg_context* ctx, const sfg_tensor* src, const sfg_format* dst, sfg_tensor** out);

/* decompose (decompose.hpp:30-63) with the count rule
 * "sum(value) groupBy (d0, d1) -> (d0) with value ne 0 -> 1 | otherwise -> 0":
 * rows whose nonzero count >= min_sum go to *selected, the rest to
 * *remainder, both canonical COO in input order. totals (optional, device,
 * int32[rows]) receives the row totals. */
int sfg_decompose_rows(sfg_context* ctx, const sfg_tensor* coo, int64_t min_sum,
                       sfg_tensor** selected, sfg_tensor** remainder, int32_t* totals);

/* decompose (decompose.hpp:30-63) with the block count rule
 * "sum(value) groupBy (d0, d1) -> (d0/r, d1/c) with value ne 0 -> 1 | otherwise -> 0":
 * the entries of r x c blocks holding >= min_sum nonzeros go to *selected,
 * the rest to *remainder (the split behind the hybrid BELL/COO format). */
int sfg_decompose_blocks(sfg_context* ctx, const sfg_tensor* coo, int64_t r, int64_t c, int64_t min_sum,
                         sfg_tensor** selected, sfg_tensor** remainder);

/* Materialized arrays (device pointers, valid while the tensor lives). */
int sfg_tensor_view_get(sfg_context* ctx, const sfg_tensor* t, sfg_tensor_view* out);
int sfg_tensor_free(sfg_tensor* t);

/* ---------------------------------------------------------------- compute */
enum {
  SFG_COMPUTE_HOST = 1, /* x/b are host inputs and y/c host outputs (copied) */
  SFG_COMPUTE_ACCUMULATE = 2, /* y += A x instead of y = A x */
};

/* run_kernel(spmv_kernel(), {A, x}) (kernel.hpp:236-384, 32-40):
 * y[M] = A x[N], fp32 accumulate; padded slots are walked like the
 * reference (0 * x[col]); BCSR slots past M/N are guarded out. */
int sfg_spmv(sfg_context* ctx, const sfg_tensor* a, const float* x, float* y, uint32_t flags);

/* run_kernel(spmm_kernel(), {A, B}) (kernel.hpp:42-51): C[M x nd] = A B,
 * B row-major [N x nd] (leading dim ldb) in b_dtype, C fp32 (ldc). */
int sfg_spmm(sfg_context* ctx, const sfg_tensor* a, const void* b, int32_t b_dtype, int64_t nd,
             int64_t ldb, float* c, int64_t ldc, uint32_t flags);

/* ---------------------------------------------------------------- ingest */
/* read_matrix_market (io.hpp:50-121) + from_coo (tensor.hpp:118): a
 * coordinate Matrix Market file (real | integer | pattern, general |
 * symmetric) parsed on the device into a canonical COO. Same header checks
 * (SFG_ERR_UNSUPPORTED_HEADER), the same "path:line: msg" SFG_ERR_PARSE
 * errors, SFG_ERR_IO when unreadable; flags: SFG_FLAG_SUM_DUPLICATES. */
int sfg_read_matrix_market(sfg_context* ctx, const char* path, uint32_t flags, sfg_tensor** out);

/* USPT binary container (io.hpp:202-334): write_container of the tensor's
 * materialized levels (byte-identical to the reference's for the same
 * tensor) and read_container into a device tensor of the given format
 * (the container does not name its format; its level kinds must match;
 * fmt == NULL infers it from them, CSR for the CSR/CSC look-alikes).
 * SFG_ERR_IO for unreadable / truncated / bad-magic files. */
int sfg_write_container(sfg_context* ctx, const sfg_tensor* t, const char* path);
int sfg_read_container(sfg_context* ctx, const char* path, const sfg_format* fmt, sfg_tensor** out);

/* run_kernel(spgemm_kernel(), {A, B}) (kernel.hpp:53, 424-567): dense
 * C[M x N2] (fp32, ldc) = A B for two sparse operands in COO / CSR / DCSR /
 * CSC / BCSR (ELL, hybrid: SFG_ERR_UNSUPPORTED_SOURCE). flags:
 * SFG_COMPUTE_ACCUMULATE adds into C; SFG_COMPUTE_HOST: c is host memory. */
int sfg_spgemm(sfg_context* ctx, const sfg_tensor* a, const sfg_tensor* b, float* c, int64_t ldc,
               uint32_t flags);

/* ------------------------------------------------------ row partitioning */
/* nnz-balanced contiguous row split for P devices: bounds[0..P]
 * with bounds[0] = 0, bounds[P] = rows, boundaries at ptr quantiles. */
int sfg_row_partition(sfg_context* ctx, const sfg_tensor* coo, int32_t parts, int64_t* bounds);
/* The same boundary rule over a host array of the row-sorted COO's rows
 * (no device work: callers that hold the rows on the host, e.g. a launcher
 * planning the split before any GPU is touched). */
int sfgx_row_bounds_host(const int32_t* rows, int64_t nnz, int64_t n_rows, int32_t parts, int64_t* bounds);
/* Rows [r0, r1) of a canonical COO as a new COO with rows rebased to 0. */
int sfg_coo_slice_rows(sfg_context* ctx, const sfg_tensor* coo, int64_t r0, int64_t r1,
                       sfg_tensor** out);

/* Row-partitioned SpMV / SpMM over P GPUs, one process per GPU (
 * the §8b `sfg_rowpart_spmm(ctxs[], P, ncclComm_t[], ..., gather_flag)`
 * entry, one call per rank). Rank r holds its row block of A (above, then
 * converted to any format) and a replica of x / B; the output buffer holds
 * P equal chunks of chunk_rows rows (chunk_rows >= every rank's block
 * rows, e.g. the maximum over ranks). The product goes straight into chunk
 * r; with SFG_ROWPART_GATHER an in-place NCCL all-gather then completes
 * every chunk on every rank. Rows of a chunk past its block are padding.
 * The reference has no multi-device path; its run_kernel threads split a
 * single host's work (kernel.hpp:365-384).
 *
 * Communicators: rank 0 calls sfg_comm_unique_id and hands the bytes to
 * every rank (any side channel), then each rank calls sfg_comm_create.
 * NCCL is loaded at run time (the copy already in the process first). */
#define SFG_COMM_ID_BYTES 128
#define SFG_ROWPART_GATHER 1u
int sfg_comm_unique_id(uint8_t id[SFG_COMM_ID_BYTES]);
int sfg_comm_create(sfg_context* ctx, int32_t nranks, int32_t rank, const uint8_t id[SFG_COMM_ID_BYTES],
                    sfg_comm** out);
int sfg_comm_destroy(sfg_comm* comm);
/* y: P * chunk_rows floats, device. */
int sfg_rowpart_spmv(sfg_context* ctx, sfg_comm* comm, const sfg_tensor* a_block, const float* x, float* y,
                     int64_t chunk_rows, uint32_t flags);
/* c: P * chunk_rows * nd floats (row-major, ldc = nd), device. */
int sfg_rowpart_spmm(sfg_context* ctx, sfg_comm* comm, const sfg_tensor* a_block, const void* b, int32_t b_dtype,
                     int64_t nd, int64_t ldb, float* c, int64_t chunk_rows, uint32_t flags);
/* The all-gather alone: chunk `rank` of buf (chunk_elems floats each) to
 * every rank, in place. */
int sfg_allgather_chunks(sfg_context* ctx, sfg_comm* comm, float* buf, int64_t chunk_elems);

/* ------------------------------------------- synthetic inputs (bench/test) */
/* Extension entry points (no reference equivalent): the seeded generators of
 * SURVEY §8d, bit-identical to the oracle's (csrc/synth.h). */
int sfgx_gen_uniform(sfg_context* ctx, uint64_t seed, int64_t rows, int64_t cols, int32_t per_row,
                     sfg_tensor** out);
int sfgx_gen_rmat(sfg_context* ctx, uint64_t seed, int32_t scale, int64_t edges, sfg_tensor** out);
int sfgx_gen_hypersparse(sfg_context* ctx, uint64_t seed, int64_t rows, int64_t cols,
                         int64_t draws, sfg_tensor** out);
int sfgx_gen_dense(sfg_context* ctx, uint64_t seed, int64_t count, float* out);
/* Config 4: BCSR(r,c) generated directly; block present with probability
 * thresh / 2^32; value_dtype SFG_F32 or SFG_BF16. */
int sfgx_gen_block_sparse(sfg_context* ctx, uint64_t seed, int64_t rows, int64_t cols, int32_t r,
                          int32_t c, uint32_t thresh, int32_t value_dtype, sfg_tensor** out);
/* Number of this library's kernels launched so far (bench gpu_launches). */
int64_t sfgx_launch_count(void);
/* Device buffers and stream-ordered copies for callers without a CUDA
 * runtime of their own (tests, the ctypes host). kind: 0 host->device,
 * 1 device->host (synchronizes), 2 device->device. */
int sfgx_device_alloc(sfg_context* ctx, int64_t bytes, void** out);
int sfgx_device_free(sfg_context* ctx, void* p);
int sfgx_copy(sfg_context* ctx, void* dst, const void* src, int64_t bytes, int32_t kind);

#ifdef __cplusplus
}
#endif

#endif /* SPARSEFORGE_B200_H */
