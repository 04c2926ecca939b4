/* sfo.c — CPU ORACLE (test infrastructure only; see sfo.h).
 *
 * Plain-C restatement of the reference hot path for 2-D matrices. Every
 * function cites the reference file:line it follows; paths are relative to
 * /root/reference/proj/include/sparseforge/. The algorithms are restated for
 * speed (counting sorts instead of std::map / std::set), but the outputs and
 * the f64 accumulation order are the reference's.
 */
#include "sfo.h"

#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../paper_2403_05802_b200/csrc/synth.h"

static __thread char g_err[512];

static int fail(int status, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return status;
}

const char* sfo_last_error(void) { return g_err; }

struct sfo_coo {
  int64_t m, n, nnz;
  int64_t* row;
  int64_t* col;
  double* val;
};

typedef struct {
  int flags;
  int64_t lo, hi, node_count;
  int64_t nidx, nptr;
  int64_t* idx;
  int64_t* ptr;
} sfo_level;

struct sfo_mat {
  int fmt;
  int64_t m, n, r, c;
  int nlevels;
  sfo_level lv[4];
  int64_t nval;
  double* val;
};

static void* xmalloc(size_t bytes) {
  void* p = malloc(bytes ? bytes : 1);
  if (!p) {
    fprintf(stderr, "sfo: out of memory (%zu bytes)\n", bytes);
    abort();
  }
  return p;
}

static void* xcalloc(size_t n, size_t sz) {
  void* p = calloc(n ? n : 1, sz ? sz : 1);
  if (!p) {
    fprintf(stderr, "sfo: out of memory\n");
    abort();
  }
  return p;
}

static sfo_coo* coo_alloc(int64_t m, int64_t n, int64_t nnz) {
  sfo_coo* t = (sfo_coo*)xcalloc(1, sizeof *t);
  t->m = m;
  t->n = n;
  t->nnz = nnz;
  t->row = (int64_t*)xmalloc((size_t)nnz * sizeof(int64_t));
  t->col = (int64_t*)xmalloc((size_t)nnz * sizeof(int64_t));
  t->val = (double*)xmalloc((size_t)nnz * sizeof(double));
  return t;
}

void sfo_coo_free(sfo_coo* t) {
  if (!t) return;
  free(t->row);
  free(t->col);
  free(t->val);
  free(t);
}

int64_t sfo_coo_nnz(const sfo_coo* t) { return t->nnz; }
int64_t sfo_coo_rows(const sfo_coo* t) { return t->m; }
int64_t sfo_coo_cols(const sfo_coo* t) { return t->n; }

int sfo_coo_get(const sfo_coo* t, int64_t* row, int64_t* col, double* val) {
  if (row) memcpy(row, t->row, (size_t)t->nnz * sizeof(int64_t));
  if (col) memcpy(col, t->col, (size_t)t->nnz * sizeof(int64_t));
  if (val) memcpy(val, t->val, (size_t)t->nnz * sizeof(double));
  return SFO_OK;
}

/* ---------------------------------------------------------------- sorting */

/* Stable counting sort of perm[0..n) by key[perm[i]] in [0, extent). */
static void counting_pass(const int64_t* key, int64_t extent, const int64_t* perm_in,
                          int64_t* perm_out, int64_t n) {
  int64_t* cnt = (int64_t*)xcalloc((size_t)extent + 1, sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) cnt[key[perm_in[i]] + 1]++;
  for (int64_t k = 0; k < extent; ++k) cnt[k + 1] += cnt[k];
  for (int64_t i = 0; i < n; ++i) perm_out[cnt[key[perm_in[i]]]++] = perm_in[i];
  free(cnt);
}

/* Stable merge sort of perm by (row, col); fallback for huge extents. */
static const int64_t* g_sort_row;
static const int64_t* g_sort_col;
static int less_rc(int64_t a, int64_t b) {
  if (g_sort_row[a] != g_sort_row[b]) return g_sort_row[a] < g_sort_row[b];
  return g_sort_col[a] < g_sort_col[b];
}
static void merge_sort(int64_t* p, int64_t* tmp, int64_t n) {
  if (n < 2) return;
  int64_t h = n / 2;
  merge_sort(p, tmp, h);
  merge_sort(p + h, tmp, n - h);
  int64_t i = 0, j = h, k = 0;
  while (i < h && j < n) tmp[k++] = less_rc(p[j], p[i]) ? p[j++] : p[i++];
  while (i < h) tmp[k++] = p[i++];
  while (j < n) tmp[k++] = p[j++];
  memcpy(p, tmp, (size_t)n * sizeof(int64_t));
}

/* Permutation that stably sorts entries lexicographically by (row, col):
 * sort_entries (tensor.hpp:98-114) uses std::stable_sort with a per-level
 * compare; an LSD pair of stable counting sorts gives the same order. */
static int64_t* stable_order(const int64_t* row, const int64_t* col, int64_t nnz, int64_t m,
                             int64_t n) {
  int64_t* p = (int64_t*)xmalloc((size_t)nnz * sizeof(int64_t));
  int64_t* q = (int64_t*)xmalloc((size_t)nnz * sizeof(int64_t));
  for (int64_t i = 0; i < nnz; ++i) p[i] = i;
  if (m <= (1ll << 28) && n <= (1ll << 28)) {
    counting_pass(col, n, p, q, nnz);
    counting_pass(row, m, q, p, nnz);
  } else {
    g_sort_row = row;
    g_sort_col = col;
    merge_sort(p, q, nnz);
  }
  free(q);
  return p;
}

/* LSD radix sort of 64-bit keys, 16-bit digits, skipping constant digits. */
static void radix_sort_u64(uint64_t* keys, int64_t n) {
  uint64_t* tmp = (uint64_t*)xmalloc((size_t)n * sizeof(uint64_t));
  int64_t* cnt = (int64_t*)xmalloc(65537 * sizeof(int64_t));
  for (int shift = 0; shift < 64; shift += 16) {
    memset(cnt, 0, 65537 * sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i) cnt[((keys[i] >> shift) & 0xFFFF) + 1]++;
    int constant = 0;
    for (int d = 0; d < 65536; ++d)
      if (cnt[d + 1] == n) constant = 1;
    if (constant) continue;
    for (int d = 0; d < 65536; ++d) cnt[d + 1] += cnt[d];
    for (int64_t i = 0; i < n; ++i) tmp[cnt[(keys[i] >> shift) & 0xFFFF]++] = keys[i];
    memcpy(keys, tmp, (size_t)n * sizeof(uint64_t));
  }
  free(cnt);
  free(tmp);
}

/* --------------------------------------------------------------- from_coo */

/* from_coo (tensor.hpp:118-162): range check (131-135, before sorting),
 * stable lexicographic sort (137 -> sort_entries 98-114), then duplicate
 * rejection (147-153) or summation in sorted order (154). */
int sfo_from_coo(int64_t m, int64_t n, int64_t nnz, const int64_t* row, const int64_t* col,
                 const double* val, int sum_duplicates, sfo_coo** out) {
  *out = NULL;
  if (nnz < 0) return fail(SFO_ERR_INVALID_OPERATION, "coordinate rank mismatch");
  for (int64_t e = 0; e < nnz; ++e)
    if (row[e] < 0 || row[e] >= m)
      return fail(SFO_ERR_INVALID_OPERATION, "coordinate out of range");
  for (int64_t e = 0; e < nnz; ++e)
    if (col[e] < 0 || col[e] >= n)
      return fail(SFO_ERR_INVALID_OPERATION, "coordinate out of range");
  int64_t* p = stable_order(row, col, nnz, m, n);
  sfo_coo* t = coo_alloc(m, n, nnz);
  int64_t k = 0;
  for (int64_t i = 0; i < nnz; ++i) {
    int64_t e = p[i];
    if (k > 0 && t->row[k - 1] == row[e] && t->col[k - 1] == col[e]) {
      if (!sum_duplicates) {
        int st = fail(SFO_ERR_DUPLICATE_COORDINATE, "duplicate coordinate (%lld,%lld)",
                      (long long)row[e], (long long)col[e]);
        free(p);
        sfo_coo_free(t);
        return st;
      }
      t->val[k - 1] += val[e];
      continue;
    }
    t->row[k] = row[e];
    t->col[k] = col[e];
    t->val[k] = val[e];
    ++k;
  }
  free(p);
  t->nnz = k;
  *out = t;
  return SFO_OK;
}

/* ----------------------------------------------------------- conversions */

static sfo_mat* mat_alloc(int fmt, const sfo_coo* s, int nlevels) {
  sfo_mat* a = (sfo_mat*)xcalloc(1, sizeof *a);
  a->fmt = fmt;
  a->m = s->m;
  a->n = s->n;
  a->nlevels = nlevels;
  return a;
}

static void level_set(sfo_level* l, int flags, int64_t lo, int64_t hi, int64_t nodes) {
  l->flags = flags;
  l->lo = lo;
  l->hi = hi;
  l->node_count = nodes;
}

static int64_t* dup64(const int64_t* src, int64_t n) {
  int64_t* d = (int64_t*)xmalloc((size_t)n * sizeof(int64_t));
  memcpy(d, src, (size_t)n * sizeof(int64_t));
  return d;
}

static double* dupf64(const double* src, int64_t n) {
  double* d = (double*)xmalloc((size_t)n * sizeof(double));
  memcpy(d, src, (size_t)n * sizeof(double));
  return d;
}

static int64_t floor_div64(int64_t a, int64_t b) {
  int64_t q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
  return q;
}

/* COO: empty plan; materialize gives one idx node per entry at both levels
 * (storage.hpp:142-149: L0 is neither merged nor above an all-dense tail). */
static sfo_mat* to_coo(const sfo_coo* s) {
  sfo_mat* a = mat_alloc(SFO_COO, s, 2);
  level_set(&a->lv[0], SFO_IDX, 0, s->m - 1, s->nnz);
  level_set(&a->lv[1], SFO_IDX, 0, s->n - 1, s->nnz);
  a->lv[0].nidx = a->lv[1].nidx = s->nnz;
  a->lv[0].idx = dup64(s->row, s->nnz);
  a->lv[1].idx = dup64(s->col, s->nnz);
  a->nval = s->nnz;
  a->val = dupf64(s->val, s->nnz);
  return a;
}

/* Parent pointers of a sorted key column (storage.hpp:195-199: ptr[p+1] =
 * ptr[p] + child count; parents without children keep an empty run, the
 * dangling nodes Fill leaves behind, operators.hpp:362-376). */
static int64_t* ptr_of(const int64_t* key, int64_t nnz, int64_t parents) {
  int64_t* ptr = (int64_t*)xcalloc((size_t)parents + 1, sizeof(int64_t));
  for (int64_t e = 0; e < nnz; ++e) ptr[key[e] + 1]++;
  for (int64_t p = 0; p < parents; ++p) ptr[p + 1] += ptr[p];
  return ptr;
}

/* CSR: plan Fill(0) Merge(0) (planner.hpp:242-249); storage
 * L0 size | L1 ptr, idx | val. */
static sfo_mat* to_csr(const sfo_coo* s) {
  sfo_mat* a = mat_alloc(SFO_CSR, s, 2);
  level_set(&a->lv[0], SFO_SIZE, 0, s->m - 1, s->m);
  level_set(&a->lv[1], SFO_PTR | SFO_IDX, 0, s->n - 1, s->nnz);
  a->lv[1].nptr = s->m + 1;
  a->lv[1].ptr = ptr_of(s->row, s->nnz, s->m);
  a->lv[1].nidx = s->nnz;
  a->lv[1].idx = dup64(s->col, s->nnz);
  a->nval = s->nnz;
  a->val = dupf64(s->val, s->nnz);
  return a;
}

/* CSC: plan Swap(0,1) Sort Fill(0) Merge(0). Swap exchanges the columns
 * and level metadata (operators.hpp:234-241); Sort is the stable
 * sort_entries (tensor.hpp:98) — on row-sorted input a stable counting
 * sort by column. */
static sfo_mat* to_csc(const sfo_coo* s) {
  sfo_mat* a = mat_alloc(SFO_CSC, s, 2);
  int64_t* p = (int64_t*)xmalloc((size_t)s->nnz * sizeof(int64_t));
  int64_t* q = (int64_t*)xmalloc((size_t)s->nnz * sizeof(int64_t));
  for (int64_t i = 0; i < s->nnz; ++i) p[i] = i;
  counting_pass(s->col, s->n, p, q, s->nnz);
  level_set(&a->lv[0], SFO_SIZE, 0, s->n - 1, s->n);
  level_set(&a->lv[1], SFO_PTR | SFO_IDX, 0, s->m - 1, s->nnz);
  a->lv[1].nptr = s->n + 1;
  a->lv[1].ptr = ptr_of(s->col, s->nnz, s->n);
  a->lv[1].nidx = s->nnz;
  a->lv[1].idx = (int64_t*)xmalloc((size_t)s->nnz * sizeof(int64_t));
  a->nval = s->nnz;
  a->val = (double*)xmalloc((size_t)s->nnz * sizeof(double));
  for (int64_t i = 0; i < s->nnz; ++i) {
    a->lv[1].idx[i] = s->row[q[i]];
    a->val[i] = s->val[q[i]];
  }
  free(p);
  free(q);
  return a;
}

/* DCSR: plan Merge(0); L0 idx is fused because the level is merged
 * (storage.hpp:146, 182-183): one node per distinct row. */
static sfo_mat* to_dcsr(const sfo_coo* s) {
  sfo_mat* a = mat_alloc(SFO_DCSR, s, 2);
  int64_t nnr = 0;
  for (int64_t e = 0; e < s->nnz; ++e)
    if (e == 0 || s->row[e] != s->row[e - 1]) ++nnr;
  level_set(&a->lv[0], SFO_IDX, 0, s->m - 1, nnr);
  level_set(&a->lv[1], SFO_PTR | SFO_IDX, 0, s->n - 1, s->nnz);
  a->lv[0].nidx = nnr;
  a->lv[0].idx = (int64_t*)xmalloc((size_t)nnr * sizeof(int64_t));
  a->lv[1].nptr = nnr + 1;
  a->lv[1].ptr = (int64_t*)xmalloc((size_t)(nnr + 1) * sizeof(int64_t));
  int64_t k = 0;
  for (int64_t e = 0; e < s->nnz; ++e)
    if (e == 0 || s->row[e] != s->row[e - 1]) {
      a->lv[0].idx[k] = s->row[e];
      a->lv[1].ptr[k] = e;
      ++k;
    }
  a->lv[1].ptr[nnr] = s->nnz;
  a->lv[1].nidx = s->nnz;
  a->lv[1].idx = dup64(s->col, s->nnz);
  a->nval = s->nnz;
  a->val = dupf64(s->val, s->nnz);
  return a;
}

/* ELL: plan Sum(0) Enumerate(0) Sort Fill(1,PadPath) Merge(0)
 * (planner.hpp:218-249). Sum: per-row count of value != 0 (formats.hpp:
 * 20-23, query_engine.hpp:112-125). Enumerate (query_engine.hpp:166-201,
 * formats.hpp:25-28): nonzeros of a row get 0..nz-1 in column order,
 * explicit zeros continue from nz. Fill(1, PadPath) inserts, for every slot
 * and every row without an entry in it, one path with the level-2 lower
 * bound (0) and value 0 (operators.hpp:203-226). Storage
 * L0 idx | L1 size | L2 idx | val, slot-major. */
static sfo_mat* to_ell(const sfo_coo* s) {
  sfo_mat* a = mat_alloc(SFO_ELL, s, 3);
  int64_t* slot = (int64_t*)xmalloc((size_t)s->nnz * sizeof(int64_t));
  int64_t k_slots = 0;
  for (int64_t b = 0; b < s->nnz;) {
    int64_t e = b;
    while (e < s->nnz && s->row[e] == s->row[b]) ++e;
    int64_t nz = 0;
    for (int64_t i = b; i < e; ++i) nz += s->val[i] != 0.0;
    int64_t nzr = 0, zr = 0;
    for (int64_t i = b; i < e; ++i) {
      slot[i] = s->val[i] != 0.0 ? nzr++ : nz + zr++;
      if (slot[i] + 1 > k_slots) k_slots = slot[i] + 1;
    }
    b = e;
  }
  int64_t cells = k_slots * s->m;
  /* Enumerate column bounds are [min, max] of the produced slots
   * (operators.hpp:463-469); {0, -1} when there are none. */
  level_set(&a->lv[0], SFO_IDX, 0, k_slots - 1, k_slots);
  level_set(&a->lv[1], SFO_SIZE, 0, s->m - 1, cells);
  level_set(&a->lv[2], SFO_IDX, 0, s->n - 1, cells);
  a->lv[0].nidx = k_slots;
  a->lv[0].idx = (int64_t*)xmalloc((size_t)k_slots * sizeof(int64_t));
  for (int64_t i = 0; i < k_slots; ++i) a->lv[0].idx[i] = i;
  a->lv[2].nidx = cells;
  a->lv[2].idx = (int64_t*)xcalloc((size_t)cells, sizeof(int64_t));
  a->nval = cells;
  a->val = (double*)xcalloc((size_t)cells, sizeof(double));
  for (int64_t i = 0; i < s->nnz; ++i) {
    int64_t cell = slot[i] * s->m + s->row[i];
    a->lv[2].idx[cell] = s->col[i];
    a->val[cell] = s->val[i];
  }
  free(slot);
  return a;
}

static int cmp_i64(const void* x, const void* y) {
  int64_t a = *(const int64_t*)x, b = *(const int64_t*)y;
  return (a > b) - (a < b);
}

/* BCSR(r,c): plan TileSplit(0,r) TileSplit(2,c) Swap(1,2) Sort Fill(3)
 * Fill(2) Fill(0) Vectorize(2) Merge(0). TileSplit bounds
 * (operators.hpp:263-285): div level [lo/r, hi/r]; mod level [lo%r, hi%r]
 * when the range lies in one tile, else [0, r-1] — so a single block row
 * is only M rows tall. Fill(3)/Fill(2) complete every touched block with
 * zeros, including positions past M/N (operators.hpp:346-379,203-226).
 * Storage L0 size | L1 ptr, idx | L2 size, dv | L3 size, dv | val; L1 is
 * fused (one node per block, storage.hpp:142-149). */
static sfo_mat* to_bcsr(const sfo_coo* s, int64_t r, int64_t c) {
  sfo_mat* a = mat_alloc(SFO_BCSR, s, 4);
  a->r = r;
  a->c = c;
  int64_t nbr = floor_div64(s->m - 1, r) + 1;
  int64_t nbc = floor_div64(s->n - 1, c) + 1;
  int64_t rb = (nbr == 1) ? s->m : r; /* extent of the row-in-block level */
  int64_t cb = (nbc == 1) ? s->n : c;
  /* Per block row: sorted distinct block columns. */
  int64_t* bptr = (int64_t*)xcalloc((size_t)nbr + 1, sizeof(int64_t));
  int64_t cap = 1024, nblk = 0;
  int64_t* bidx = (int64_t*)xmalloc((size_t)cap * sizeof(int64_t));
  int64_t* tmp = (int64_t*)xmalloc((size_t)(s->nnz ? s->nnz : 1) * sizeof(int64_t));
  int64_t e0 = 0;
  for (int64_t br = 0; br < nbr; ++br) {
    int64_t e1 = e0;
    while (e1 < s->nnz && s->row[e1] / r == br) ++e1;
    int64_t k = 0;
    for (int64_t e = e0; e < e1; ++e) tmp[k++] = s->col[e] / c;
    qsort(tmp, (size_t)k, sizeof(int64_t), cmp_i64);
    int64_t u = 0;
    for (int64_t i = 0; i < k; ++i)
      if (i == 0 || tmp[i] != tmp[i - 1]) tmp[u++] = tmp[i];
    if (nblk + u > cap) {
      while (nblk + u > cap) cap *= 2;
      bidx = (int64_t*)realloc(bidx, (size_t)cap * sizeof(int64_t));
    }
    memcpy(bidx + nblk, tmp, (size_t)u * sizeof(int64_t));
    nblk += u;
    bptr[br + 1] = nblk;
    e0 = e1;
  }
  free(tmp);
  level_set(&a->lv[0], SFO_SIZE, 0, nbr - 1, nbr);
  level_set(&a->lv[1], SFO_PTR | SFO_IDX, 0, nbc - 1, nblk);
  level_set(&a->lv[2], SFO_SIZE | SFO_DENSE_VECTOR, 0, rb - 1, nblk * rb);
  level_set(&a->lv[3], SFO_SIZE | SFO_DENSE_VECTOR, 0, cb - 1, nblk * rb * cb);
  a->lv[1].nptr = nbr + 1;
  a->lv[1].ptr = bptr;
  a->lv[1].nidx = nblk;
  a->lv[1].idx = bidx;
  a->nval = nblk * rb * cb;
  a->val = (double*)xcalloc((size_t)a->nval, sizeof(double));
  for (int64_t e = 0; e < s->nnz; ++e) {
    int64_t br = s->row[e] / r, bc = s->col[e] / c;
    /* binary search bc in the block row */
    int64_t lo = bptr[br], hi = bptr[br + 1] - 1;
    while (lo < hi) {
      int64_t mid = (lo + hi) / 2;
      if (bidx[mid] < bc) lo = mid + 1;
      else hi = mid;
    }
    int64_t i = s->row[e] % r, j = s->col[e] % c;
    a->val[(lo * rb + i) * cb + j] = s->val[e];
  }
  return a;
}

int sfo_convert(const sfo_coo* src, int fmt, int64_t r, int64_t c, sfo_mat** out) {
  *out = NULL;
  if (src->m <= 0 || src->n <= 0)
    return fail(SFO_ERR_INVALID_OPERATION, "empty bounds at extent-only level");
  switch (fmt) {
    case SFO_COO: *out = to_coo(src); break;
    case SFO_CSR: *out = to_csr(src); break;
    case SFO_CSC: *out = to_csc(src); break;
    case SFO_DCSR: *out = to_dcsr(src); break;
    case SFO_ELL: *out = to_ell(src); break;
    case SFO_BCSR:
      if (r <= 0 || c <= 0)
        return fail(SFO_ERR_INVALID_OPERATION, "TileSplit factor must be positive");
      *out = to_bcsr(src, r, c);
      break;
    default: return fail(SFO_ERR_PARSE, "unknown format id %d", fmt);
  }
  return SFO_OK;
}

int sfo_mat_nlevels(const sfo_mat* m) { return m->nlevels; }

int sfo_mat_level_info(const sfo_mat* m, int l, int64_t info[6]) {
  if (l < 0 || l >= m->nlevels) return fail(SFO_ERR_INVALID_OPERATION, "level out of range");
  const sfo_level* v = &m->lv[l];
  info[0] = v->flags;
  info[1] = v->lo;
  info[2] = v->hi;
  info[3] = v->node_count;
  info[4] = v->nidx;
  info[5] = v->nptr;
  return SFO_OK;
}

int sfo_mat_level_idx(const sfo_mat* m, int l, int64_t* out) {
  if (l < 0 || l >= m->nlevels) return fail(SFO_ERR_INVALID_OPERATION, "level out of range");
  if (m->lv[l].nidx) memcpy(out, m->lv[l].idx, (size_t)m->lv[l].nidx * sizeof(int64_t));
  return SFO_OK;
}

int sfo_mat_level_ptr(const sfo_mat* m, int l, int64_t* out) {
  if (l < 0 || l >= m->nlevels) return fail(SFO_ERR_INVALID_OPERATION, "level out of range");
  if (m->lv[l].nptr) memcpy(out, m->lv[l].ptr, (size_t)m->lv[l].nptr * sizeof(int64_t));
  return SFO_OK;
}

int64_t sfo_mat_nvals(const sfo_mat* m) { return m->nval; }

int sfo_mat_values(const sfo_mat* m, double* out) {
  if (m->nval) memcpy(out, m->val, (size_t)m->nval * sizeof(double));
  return SFO_OK;
}

void sfo_mat_free(sfo_mat* m) {
  if (!m) return;
  for (int l = 0; l < m->nlevels; ++l) {
    free(m->lv[l].idx);
    free(m->lv[l].ptr);
  }
  free(m->val);
  free(m);
}

/* ---------------------------------------------------------------- kernels */

/* run_kernel, single sparse operand, optimize on (kernel.hpp:339-364): walk
 * every stored slot in storage order (walk_slots, storage.hpp:238-280),
 * padding included; restore logical (d0, d1) through the inverse map;
 * skip slots failing the bounds guard (kernel.hpp:290-302); accumulate
 * prod = value * dense(...) into the output cell (kernel.hpp:274-286).
 * visit(row, col, slot) is called in exactly that order. */
typedef void (*slot_fn)(void* ctx, int64_t row, int64_t col, double v);

static void walk(const sfo_mat* a, slot_fn fn, void* ctx) {
  switch (a->fmt) {
    case SFO_COO:
      for (int64_t k = 0; k < a->nval; ++k) fn(ctx, a->lv[0].idx[k], a->lv[1].idx[k], a->val[k]);
      break;
    case SFO_CSR:
      for (int64_t r = 0; r < a->m; ++r)
        for (int64_t k = a->lv[1].ptr[r]; k < a->lv[1].ptr[r + 1]; ++k)
          fn(ctx, r, a->lv[1].idx[k], a->val[k]);
      break;
    case SFO_CSC: /* physical (d1, d0) restores to (d0, d1) */
      for (int64_t c = 0; c < a->n; ++c)
        for (int64_t k = a->lv[1].ptr[c]; k < a->lv[1].ptr[c + 1]; ++k)
          fn(ctx, a->lv[1].idx[k], c, a->val[k]);
      break;
    case SFO_DCSR:
      for (int64_t p = 0; p < a->lv[0].nidx; ++p)
        for (int64_t k = a->lv[1].ptr[p]; k < a->lv[1].ptr[p + 1]; ++k)
          fn(ctx, a->lv[0].idx[p], a->lv[1].idx[k], a->val[k]);
      break;
    case SFO_ELL: /* (slot, d0, d1) restores to (d0, d1) */
      for (int64_t s = 0; s < a->lv[0].nidx; ++s)
        for (int64_t r = 0; r < a->m; ++r) {
          int64_t cell = s * a->m + r;
          fn(ctx, r, a->lv[2].idx[cell], a->val[cell]);
        }
      break;
    case SFO_BCSR: {
      int64_t rb = a->lv[2].hi - a->lv[2].lo + 1, cb = a->lv[3].hi - a->lv[3].lo + 1;
      for (int64_t br = 0; br < a->lv[0].node_count; ++br)
        for (int64_t k = a->lv[1].ptr[br]; k < a->lv[1].ptr[br + 1]; ++k)
          for (int64_t i = 0; i < rb; ++i)
            for (int64_t j = 0; j < cb; ++j) {
              /* inverse of (d0/r, d1/c, d0%r, d1%c) */
              int64_t row = br * a->r + a->lv[2].lo + i, col = a->lv[1].idx[k] * a->c + a->lv[3].lo + j;
              if (row >= a->m || col >= a->n) continue; /* bounds guard */
              fn(ctx, row, col, a->val[(k * rb + i) * cb + j]);
            }
      break;
    }
  }
}

typedef struct {
  const double* x;
  double* y;
} spmv_ctx;

static void spmv_visit(void* p, int64_t row, int64_t col, double v) {
  spmv_ctx* c = (spmv_ctx*)p;
  c->y[row] += v * c->x[col];
}

int sfo_spmv(const sfo_mat* a, const double* x, double* y) {
  memset(y, 0, (size_t)a->m * sizeof(double));
  spmv_ctx c = {x, y};
  walk(a, spmv_visit, &c);
  return SFO_OK;
}

typedef struct {
  const double* b;
  double* c;
  int64_t nd;
} spmm_ctx;

static void spmm_visit(void* p, int64_t row, int64_t col, double v) {
  spmm_ctx* c = (spmm_ctx*)p;
  const double* brow = c->b + col * c->nd;
  double* crow = c->c + row * c->nd;
  for (int64_t j = 0; j < c->nd; ++j) crow[j] += v * brow[j];
}

int sfo_spmm(const sfo_mat* a, const double* b, int64_t nd, double* c) {
  memset(c, 0, (size_t)(a->m * nd) * sizeof(double));
  spmm_ctx x = {b, c, nd};
  walk(a, spmm_visit, &x);
  return SFO_OK;
}

/* -------------------------------------------------------------- decompose */

/* decompose (decompose.hpp:30-63): group totals over the dense row domain
 * (query_engine.hpp:112-125 with dense_group_keys 57-77), then each entry
 * goes to `selected` when its group's total >= min_sum (decompose.hpp:58),
 * otherwise to `remainder`, keeping order. */
int sfo_decompose_rows(const sfo_coo* t, int64_t min_sum, sfo_coo** selected,
                       sfo_coo** remainder, int64_t* totals_out) {
  int64_t* tot = (int64_t*)xcalloc((size_t)t->m, sizeof(int64_t));
  for (int64_t e = 0; e < t->nnz; ++e) tot[t->row[e]] += t->val[e] != 0.0;
  int64_t nsel = 0;
  for (int64_t e = 0; e < t->nnz; ++e) nsel += tot[t->row[e]] >= min_sum;
  sfo_coo* s = coo_alloc(t->m, t->n, nsel);
  sfo_coo* r = coo_alloc(t->m, t->n, t->nnz - nsel);
  int64_t a = 0, b = 0;
  for (int64_t e = 0; e < t->nnz; ++e) {
    if (tot[t->row[e]] >= min_sum) {
      s->row[a] = t->row[e];
      s->col[a] = t->col[e];
      s->val[a++] = t->val[e];
    } else {
      r->row[b] = t->row[e];
      r->col[b] = t->col[e];
      r->val[b++] = t->val[e];
    }
  }
  if (totals_out) memcpy(totals_out, tot, (size_t)t->m * sizeof(int64_t));
  free(tot);
  *selected = s;
  *remainder = r;
  return SFO_OK;
}

/* ------------------------------------------------------------- generators */

int sfo_gen_uniform(uint64_t seed, int64_t m, int64_t n, int per_row, sfo_coo** out) {
  if (per_row > n || per_row > 64) return fail(SFO_ERR_INVALID_OPERATION, "per_row too large");
  sfo_coo* t = coo_alloc(m, n, m * per_row);
  uint32_t cols[64];
  for (int64_t r = 0; r < m; ++r) {
    sfg_uniform_row(seed, (uint32_t)r, (uint32_t)n, per_row, cols);
    for (int i = 0; i < per_row; ++i) {
      int64_t e = r * per_row + i;
      t->row[e] = r;
      t->col[e] = cols[i];
      t->val[e] = (double)sfg_coord_value(seed, (uint32_t)r, cols[i]);
    }
  }
  *out = t;
  return SFO_OK;
}

static sfo_coo* from_keys(uint64_t seed, uint64_t* keys, int64_t n, int64_t m, int64_t ncols) {
  radix_sort_u64(keys, n);
  int64_t u = 0;
  for (int64_t i = 0; i < n; ++i)
    if (i == 0 || keys[i] != keys[i - 1]) keys[u++] = keys[i];
  sfo_coo* t = coo_alloc(m, ncols, u);
  for (int64_t i = 0; i < u; ++i) {
    uint32_t r = (uint32_t)(keys[i] >> 32), c = (uint32_t)keys[i];
    t->row[i] = r;
    t->col[i] = c;
    t->val[i] = (double)sfg_coord_value(seed, r, c);
  }
  return t;
}

int sfo_gen_rmat(uint64_t seed, int scale, int64_t edges, sfo_coo** out) {
  uint64_t* keys = (uint64_t*)xmalloc((size_t)edges * sizeof(uint64_t));
  for (int64_t e = 0; e < edges; ++e) keys[e] = sfg_rmat_edge(seed, (uint64_t)e, scale);
  *out = from_keys(seed, keys, edges, 1ll << scale, 1ll << scale);
  free(keys);
  return SFO_OK;
}

int sfo_gen_hypersparse(uint64_t seed, int64_t m, int64_t n, int64_t draws, sfo_coo** out) {
  uint64_t* keys = (uint64_t*)xmalloc((size_t)draws * sizeof(uint64_t));
  for (int64_t k = 0; k < draws; ++k)
    keys[k] = sfg_uniform_coord(seed, (uint64_t)k, (uint32_t)m, (uint32_t)n);
  *out = from_keys(seed, keys, draws, m, n);
  free(keys);
  return SFO_OK;
}

/* COO expansion of the config-4 block-sparse matrix, (row, col)-sorted. */
int sfo_gen_block_sparse(uint64_t seed, int64_t m, int64_t n, int64_t r, int64_t c, uint32_t thresh,
                         sfo_coo** out) {
  int64_t nbr = (m - 1) / r + 1, nbc = (n - 1) / c + 1, cnt = 0;
  for (int64_t br = 0; br < nbr; ++br)
    for (int64_t bc = 0; bc < nbc; ++bc)
      if (sfg_block_present(seed, (uint32_t)br, (uint32_t)bc, thresh)) {
        int64_t rows = (br + 1) * r <= m ? r : m - br * r, cols = (bc + 1) * c <= n ? c : n - bc * c;
        cnt += rows * cols;
      }
  sfo_coo* t = coo_alloc(m, n, cnt);
  int64_t k = 0;
  for (int64_t row = 0; row < m; ++row) {
    int64_t br = row / r;
    for (int64_t bc = 0; bc < nbc; ++bc) {
      if (!sfg_block_present(seed, (uint32_t)br, (uint32_t)bc, thresh)) continue;
      for (int64_t col = bc * c; col < (bc + 1) * c && col < n; ++col) {
        t->row[k] = row;
        t->col[k] = col;
        t->val[k++] = (double)sfg_coord_value(seed, (uint32_t)row, (uint32_t)col);
      }
    }
  }
  *out = t;
  return SFO_OK;
}

void sfo_gen_dense(uint64_t seed, int64_t count, double* out) {
  for (int64_t i = 0; i < count; ++i)
    out[i] = (double)sfg_dense_value(sfg_hash3(seed, (uint64_t)i, 0x77));
}
