/* oracle.c -- TEST INFRASTRUCTURE ONLY.  The plain, slow, obviously-correct CPU KNN join that the CUDA
 * path is checked against.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this.  It shares no code, header, table or helper with
 * paper_1011_2807_b200/ (the product path); neither side includes or links the other.
 *
 * What it computes (the plain definition, §3):
 *   for every r in R (in the given row order) and every s in S (ascending id):
 *     v = dot(r, s) = sum_i r[i]*s[i]                             (Eq. 1)
 *       evaluated with the two-iterator merge of Alg. 2 lines 8-23;
 *       fp64 accumulation for fp32 inputs (every fp32 x {1, int8, fp32} product is exact in fp64),
 *       int64 accumulation for integer (binary / int8) inputs.
 *     keep (v, s) iff v > 0   (zero scores are never admitted: pruneScore starts at 0 and the test is
 *                              strict; reading c2)
 *   sort the kept pairs by (v descending, s ascending)  (reading c1: ties to the lower S id,
 *                              BASELINE.json north_star "tie-break on lower S id")
 *   emit the first k; pad with (id -1, score 0) to length k (reading c2).
 * Single-threaded; a library sort (qsort) is the only primitive used.
 *
 * dtype codes: 0 = binary (values == NULL, every weight is 1), 1 = int8, 2 = fp32.
 */
#include <stdint.h>
#include <stdlib.h>

typedef struct {
  int64_t n_rows;
  const int64_t* indptr;
  const int32_t* indices;
  const void* values;
  int32_t dtype;
} ocsr;

static double wval(const ocsr* m, int64_t p) {
  if (m->dtype == 0) return 1.0;
  if (m->dtype == 1) return (double)((const int8_t*)m->values)[p];
  return (double)((const float*)m->values)[p];
}
static int64_t ival(const ocsr* m, int64_t p) {
  if (m->dtype == 0) return 1;
  return (int64_t)((const int8_t*)m->values)[p];
}

/* dot(r, s): Alg. 2 lines 8-23, the two-pointer merge over ascending features.  `advances`, if not NULL,
 * receives the number of iterator advances (SPEC.md:58 feature_visits; <= |r|+|s|, Eq. 2). */
double oracle_dot(const ocsr* R, int64_t r, const ocsr* S, int64_t s, int64_t* advances) {
  int64_t i = R->indptr[r], ie = R->indptr[r + 1];
  int64_t j = S->indptr[s], je = S->indptr[s + 1];
  int integer = (R->dtype != 2 && S->dtype != 2);
  double ret = 0.0;
  int64_t iret = 0, adv = 0;
  while (i < ie && j < je) {
    int32_t dr = R->indices[i], ds = S->indices[j];
    if (dr == ds) {
      if (integer) iret += ival(R, i) * ival(S, j);
      else ret += wval(R, i) * wval(S, j);
      ++i; ++j; adv += 2;
    } else if (dr > ds) {
      ++j; ++adv;
    } else {
      ++i; ++adv;
    }
  }
  if (advances) *advances += adv;
  return integer ? (double)iret : ret;
}

typedef struct { double v; int64_t s; } cand;

static int cand_cmp(const void* a, const void* b) {
  const cand* x = (const cand*)a;
  const cand* y = (const cand*)b;
  if (x->v > y->v) return -1;
  if (x->v < y->v) return 1;
  return (x->s > y->s) - (x->s < y->s);
}

/* The oracle: rows `rows[0..n_sel)` of R (all rows if rows == NULL, n_sel = R->n_rows) against every row
 * of S.  out_ids[n_sel*k] (S id + s_id_base, or -1), out_scores[n_sel*k] (exact fp64 / integer value, or
 * 0).  Returns 0, or 1 on allocation failure. */
int oracle_knn(const ocsr* R, const ocsr* S, const int64_t* rows, int64_t n_sel, int32_t k, int64_t s_id_base,
               int64_t* out_ids, double* out_scores) {
  cand* buf = (cand*)malloc(sizeof(cand) * (size_t)(S->n_rows > 0 ? S->n_rows : 1));
  if (!buf) return 1;
  for (int64_t q = 0; q < n_sel; ++q) {
    int64_t r = rows ? rows[q] : q;
    int64_t m = 0;
    for (int64_t s = 0; s < S->n_rows; ++s) {
      double v = oracle_dot(R, r, S, s, NULL);
      if (v > 0.0) { buf[m].v = v; buf[m].s = s; ++m; }
    }
    qsort(buf, (size_t)m, sizeof(cand), cand_cmp);
    for (int32_t t = 0; t < k; ++t) {
      if (t < m) {
        out_ids[q * k + t] = buf[t].s + s_id_base;
        out_scores[q * k + t] = buf[t].v;
      } else {
        out_ids[q * k + t] = -1;
        out_scores[q * k + t] = 0.0;
      }
    }
  }
  free(buf);
  return 0;
}

/* Exact scores of given (r, s) pairs, used to evaluate the tolerance rule on fp32 configs (DESIGN.md
 * reading c15: x(g_i) is the oracle's exact score of the GPU's id). */
void oracle_pair_scores(const ocsr* R, const ocsr* S, const int64_t* r_rows, const int64_t* s_rows, int64_t n,
                        double* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = (s_rows[i] < 0) ? 0.0 : oracle_dot(R, r_rows[i], S, s_rows[i], NULL);
}

/* Eq. 3 counter: BF charges |r|+|s| per pair; also returns the true merge advances. */
void oracle_bf_counters(const ocsr* R, const ocsr* S, int64_t* charged, int64_t* advances) {
  int64_t c = 0, a = 0;
  for (int64_t r = 0; r < R->n_rows; ++r)
    for (int64_t s = 0; s < S->n_rows; ++s) {
      c += (R->indptr[r + 1] - R->indptr[r]) + (S->indptr[s + 1] - S->indptr[s]);
      oracle_dot(R, r, S, s, &a);
    }
  *charged = c;
  *advances = a;
}
