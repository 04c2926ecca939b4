/* sfo — CPU ORACLE (test infrastructure only).
 *
 * A plain-C restatement of the reference's hot path (sparse-forge,
 * /root/reference/proj/include/sparseforge) for 2-D matrices: from_coo,
 * the COO -> {COO, CSR, CSC, DCSR, ELL, BCSR(r,c)} conversions as they come
 * out of plan_conversion + apply_plan + materialize, the row-count
 * decompose, and run_kernel's single-sparse-operand SpMV/SpMM walk.
 * Indices are int64 and values f64, exactly like the reference.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library, and only as the checker.
 * It is pinned against the reference's own golden vectors
 * (proj/tests/oracle_data.hpp, via tests/golden/) and against the reference
 * headers compiled unmodified (oracle/_ref/libsfref.so, oracle/ref_shim.cpp).
 */
#ifndef SFO_H
#define SFO_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status: 0 = ok, otherwise 1 + the reference ErrorKind ordinal
 * (errors.hpp:10-21). */
enum {
  SFO_OK = 0,
  SFO_ERR_PARSE = 1,
  SFO_ERR_NON_AFFINE = 2,
  SFO_ERR_NON_INTEGRAL = 3,
  SFO_ERR_UNSUPPORTED_SOURCE = 4,
  SFO_ERR_UNSUPPORTED_HEADER = 5,
  SFO_ERR_DUPLICATE_COORDINATE = 6,
  SFO_ERR_COLLISION = 7,
  SFO_ERR_INVALID_OPERATION = 8,
  SFO_ERR_SINGULAR = 9,
  SFO_ERR_IO = 10,
};

enum { SFO_COO = 0, SFO_CSR = 1, SFO_CSC = 2, SFO_DCSR = 3, SFO_ELL = 4, SFO_BCSR = 5 };

/* LevelStorage flags (storage.hpp:17-22). */
enum { SFO_SIZE = 1, SFO_PTR = 2, SFO_IDX = 4, SFO_DENSE_VECTOR = 8 };

typedef struct sfo_coo sfo_coo;
typedef struct sfo_mat sfo_mat;

const char* sfo_last_error(void);

/* from_coo (tensor.hpp:118-162). */
int sfo_from_coo(int64_t m, int64_t n, int64_t nnz, const int64_t* row, const int64_t* col,
                 const double* val, int sum_duplicates, sfo_coo** out);
int64_t sfo_coo_nnz(const sfo_coo* t);
int64_t sfo_coo_rows(const sfo_coo* t);
int64_t sfo_coo_cols(const sfo_coo* t);
int sfo_coo_get(const sfo_coo* t, int64_t* row, int64_t* col, double* val);
void sfo_coo_free(sfo_coo* t);

/* convert_structure(COO -> fmt) + materialize(infer_storage(fmt))
 * (planner.hpp:261-265, storage.hpp:97-234). r, c: BCSR block shape. */
int sfo_convert(const sfo_coo* src, int fmt, int64_t r, int64_t c, sfo_mat** out);
int sfo_mat_nlevels(const sfo_mat* m);
/* info = {flags, bounds.lo, bounds.hi, node_count, len(idx), len(ptr)} */
int sfo_mat_level_info(const sfo_mat* m, int level, int64_t info[6]);
int sfo_mat_level_idx(const sfo_mat* m, int level, int64_t* out);
int sfo_mat_level_ptr(const sfo_mat* m, int level, int64_t* out);
int64_t sfo_mat_nvals(const sfo_mat* m);
int sfo_mat_values(const sfo_mat* m, double* out);
void sfo_mat_free(sfo_mat* m);

/* run_kernel single-sparse path (kernel.hpp:339-364): y = A x,
 * C[M x nd] = A B[N x nd], row-major, outputs overwritten. */
int sfo_spmv(const sfo_mat* a, const double* x, double* y);
int sfo_spmm(const sfo_mat* a, const double* b, int64_t nd, double* c);

/* decompose (decompose.hpp:30-63) with the count rule
 * sum(value) groupBy (d0, d1) -> (d0) with value ne 0 -> 1 | otherwise -> 0.
 * totals (optional) receives the M row totals. */
int sfo_decompose_rows(const sfo_coo* t, int64_t min_sum, sfo_coo** selected,
                       sfo_coo** remainder, int64_t* totals);

/* Synthetic inputs, identical to the GPU generators. */
int sfo_gen_uniform(uint64_t seed, int64_t m, int64_t n, int per_row, sfo_coo** out);
int sfo_gen_rmat(uint64_t seed, int scale, int64_t edges, sfo_coo** out);
int sfo_gen_hypersparse(uint64_t seed, int64_t m, int64_t n, int64_t draws, sfo_coo** out);
void sfo_gen_dense(uint64_t seed, int64_t count, double* out);
int sfo_gen_block_sparse(uint64_t seed, int64_t m, int64_t n, int64_t r, int64_t c, uint32_t thresh,
                         sfo_coo** out);

#ifdef __cplusplus
}
#endif

#endif /* SFO_H */
