/* iib.c -- TEST / BENCH INFRASTRUCTURE ONLY.  The paper's IIB algorithm (Alg. 3) on the host
 * CPU, single-threaded, as the "paper's method on the host" baseline of bench.py.  Only
 * tests/ and bench.py's cpu_baseline leg load it; it shares nothing with paper_1011_2807_b200/.
 *
 *   Create_Inverted_List_IIB (Alg. 3 lines 5-8): for every s of S (ascending) and every
 *     feature (d, w) of s, append (s, w) to I_d  -- here a CSC built by counting sort, so each I_d is ascending s.
 *   Find_Matches_IIB (lines 9-17), for every r:
 *     A[s] += r[d] * w for every (s, w) in I_d, for every (d, r[d]) of r     (the accumulator A, line 12)
 *     every s with A[s] > 0 is a candidate; keep the k best by (score desc, id asc)  (lines 14-16, reading c1)
 *   fp64 accumulation for fp32 inputs, int64 for integer ones (as the oracle); A is a dense array with a list of
 *   touched ids (reset after each r), the candidate set a sorted insertion list of k entries.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int64_t n_rows;
  const int64_t* indptr;
  const int32_t* indices;
  const void* values;
  int32_t dtype; /* 0 binary, 1 int8, 2 fp32 */
} icsr;

typedef struct {
  int32_t d;
  int64_t n_s;
  int64_t* ptr;   /* [d + 1] */
  int32_t* sid;   /* [nnz] S row of each posting */
  double* w;      /* [nnz] weight of each posting */
} iib_index;

static double wv(const icsr* m, int64_t p) {
  if (m->dtype == 0) return 1.0;
  if (m->dtype == 1) return (double)((const int8_t*)m->values)[p];
  return (double)((const float*)m->values)[p];
}

/* Alg. 3 lines 5-8.  Returns NULL on allocation failure. */
iib_index* iib_build(const icsr* S, int32_t d) {
  iib_index* ix = (iib_index*)calloc(1, sizeof(iib_index));
  if (!ix) return NULL;
  const int64_t nnz = S->indptr[S->n_rows];
  ix->d = d;
  ix->n_s = S->n_rows;
  ix->ptr = (int64_t*)calloc((size_t)d + 1, sizeof(int64_t));
  ix->sid = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nnz > 0 ? nnz : 1));
  ix->w = (double*)malloc(sizeof(double) * (size_t)(nnz > 0 ? nnz : 1));
  if (!ix->ptr || !ix->sid || !ix->w) return NULL;
  for (int64_t j = 0; j < nnz; ++j)
    if (S->indices[j] >= 0 && S->indices[j] < d) ix->ptr[S->indices[j] + 1]++;
  for (int32_t f = 0; f < d; ++f) ix->ptr[f + 1] += ix->ptr[f];
  int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)(d > 0 ? d : 1));
  if (!fill) return NULL;
  memcpy(fill, ix->ptr, sizeof(int64_t) * (size_t)d);
  for (int64_t s = 0; s < S->n_rows; ++s)
    for (int64_t j = S->indptr[s]; j < S->indptr[s + 1]; ++j) {
      const int32_t f = S->indices[j];
      if (f < 0 || f >= d) continue;
      const int64_t at = fill[f]++;
      ix->sid[at] = (int32_t)s;
      ix->w[at] = wv(S, j);
    }
  free(fill);
  return ix;
}

void iib_free(iib_index* ix) {
  if (!ix) return;
  free(ix->ptr);
  free(ix->sid);
  free(ix->w);
  free(ix);
}

/* Alg. 3 lines 9-17 for rows rows[0..n_sel) of R.  out_ids (S id or -1), out_scores (or 0).  visits (optional)
 * receives the number of postings accumulated (Eq. 4's second term).  Returns 0 or 1 (alloc). */
int iib_query(const iib_index* ix, const icsr* R, const int64_t* rows, int64_t n_sel, int32_t k, int64_t* out_ids,
              double* out_scores, int64_t* visits) {
  double* A = (double*)calloc((size_t)(ix->n_s > 0 ? ix->n_s : 1), sizeof(double));
  int32_t* touched = (int32_t*)malloc(sizeof(int32_t) * (size_t)(ix->n_s > 0 ? ix->n_s : 1));
  double* cs = (double*)malloc(sizeof(double) * (size_t)k);
  int64_t* ci = (int64_t*)malloc(sizeof(int64_t) * (size_t)k);
  if (!A || !touched || !cs || !ci) return 1;
  int64_t v = 0;
  for (int64_t q = 0; q < n_sel; ++q) {
    const int64_t r = rows ? rows[q] : q;
    int64_t nt = 0;
    for (int64_t j = R->indptr[r]; j < R->indptr[r + 1]; ++j) {
      const int32_t f = R->indices[j];
      if (f < 0 || f >= ix->d) continue;
      const double rv = wv(R, j);
      for (int64_t p = ix->ptr[f]; p < ix->ptr[f + 1]; ++p) {
        const int32_t s = ix->sid[p];
        if (A[s] == 0.0) touched[nt++] = s;
        A[s] += rv * ix->w[p];
      }
      v += ix->ptr[f + 1] - ix->ptr[f];
    }
    /* candidate set (lines 14-16): sorted list of at most k (score desc, id asc); strict admission */
    int32_t m = 0;
    for (int64_t t = 0; t < nt; ++t) {
      const int32_t s = touched[t];
      const double x = A[s];
      A[s] = 0.0;
      if (!(x > 0.0)) continue;
      if (m == k && !(x > cs[k - 1] || (x == cs[k - 1] && s < ci[k - 1]))) continue;
      int32_t pos = m < k ? m : k - 1;
      while (pos > 0 && (cs[pos - 1] < x || (cs[pos - 1] == x && ci[pos - 1] > s))) {
        cs[pos] = cs[pos - 1];
        ci[pos] = ci[pos - 1];
        --pos;
      }
      cs[pos] = x;
      ci[pos] = s;
      if (m < k) ++m;
    }
    for (int32_t i = 0; i < k; ++i) {
      out_ids[q * k + i] = i < m ? ci[i] : -1;
      out_scores[q * k + i] = i < m ? cs[i] : 0.0;
    }
  }
  if (visits) *visits += v;
  free(A);
  free(touched);
  free(cs);
  free(ci);
  return 0;
}
