/* gen.c -- seeded synthetic CSR generator for the five BASELINE.json configs (SURVEY.md §8 row a0,
 * recipe in §8(d) "Synthetic inputs" and DESIGN.md "Input recipe").
 *
 * This module is shared by the oracle side and the CUDA side as INPUT ONLY: it draws rows and holds
 * none of the join's arithmetic (no dot products, no top-k, no index).  Every row is a pure function
 * of (seed, config_id, set_id, row): a SplitMix64 stream keyed by those four values, so any row range
 * (an S shard on rank p, an oracle row sample) regenerates bit-identically on its own, on any thread
 * count.
 *
 * Per row, in stream order:
 *   1. count  : count_law 0 -> lo + floor(u*(hi-lo+1));  count_law 1 -> 2*(L-1), L = lo + floor(u*(hi-lo+1))
 *               (the b-/y-ion peak count of a length-L peptide, BASELINE.json configs[2]).
 *   2. features, drawn one at a time, duplicates re-drawn (rejection), then sorted ascending:
 *               feat_law 0 uniform floor(u*d); 1 Zipf(a): rank i in 1..d with P ∝ i^-a by inverse CDF on
 *               an fp64 table, feature = i-1; 2 Gaussian bands: band j = floor(u*nb), x = c_j + sigma*z,
 *               c_j = (2j+1)*d/(2nb), bin = floor(x), out-of-range re-drawn.
 *   3. values, one per feature in ascending-feature order:
 *               value_law 0 binary (no values array); 1 lognormal exp(z) cast to fp32;
 *               2 lognormal normalised to unit L2 in fp64, then cast to fp32; 3 int8 lo + floor(u*(hi-lo+1)).
 *   u = (next>>11)*2^-53 in [0,1); z = Box-Muller cos branch from two uniforms.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int64_t n_rows;
  int32_t d;
  int32_t count_law, nnz_lo, nnz_hi;
  int32_t feat_law;
  double zipf_a;
  int32_t n_bands;
  double band_sigma;
  int32_t value_law, val_lo, val_hi;
  uint64_t seed;
  uint32_t config_id, set_id;
} gen_spec;

typedef struct { uint64_t x; } rng_t;

static uint64_t splitmix_next(rng_t* r) {
  uint64_t z = (r->x += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
static uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
static rng_t row_rng(const gen_spec* g, int64_t row) {
  rng_t r;
  uint64_t k = mix64(g->seed + 0x632BE59BD9B4E019ULL);
  k = mix64(k ^ ((uint64_t)g->config_id * 0x9E3779B97F4A7C15ULL));
  k = mix64(k ^ ((uint64_t)g->set_id * 0xD1B54A32D192ED03ULL));
  k = mix64(k ^ ((uint64_t)row * 0xABC98388FB8FAC03ULL));
  r.x = k;
  return r;
}
static double unif(rng_t* r) { return (double)(splitmix_next(r) >> 11) * (1.0 / 9007199254740992.0); }
static double normal(rng_t* r) {
  double u1 = 1.0 - unif(r); /* (0,1] */
  double u2 = unif(r);
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925286766559 * u2);
}

static int32_t draw_count(const gen_spec* g, rng_t* r) {
  int32_t span = g->nnz_hi - g->nnz_lo + 1;
  int32_t c = g->nnz_lo + (int32_t)(unif(r) * span);
  if (g->count_law == 1) c = 2 * (c - 1);
  if (c > g->d) c = g->d;
  if (c < 0) c = 0;
  return c;
}

int gen_row_counts(const gen_spec* g, int64_t row0, int64_t n, int32_t* counts) {
  if (!g || g->d <= 0 || g->nnz_lo < 0 || g->nnz_hi < g->nnz_lo) return 1;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    rng_t r = row_rng(g, row0 + i);
    counts[i] = draw_count(g, &r);
  }
  return 0;
}

static int cmp_i32(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

/* Fill rows [row0, row0+n): indptr is LOCAL (indptr[0] = 0, indptr[n] = total) and must have been
 * built from gen_row_counts.  values: float* for value_law 1/2, int8_t* for 3, ignored for 0. */
int gen_fill(const gen_spec* g, int64_t row0, int64_t n, const int64_t* indptr, int32_t* indices, void* values) {
  if (!g || g->d <= 0) return 1;
  const int32_t d = g->d;
  double* cdf = NULL;
  if (g->feat_law == 1) {
    cdf = (double*)malloc(sizeof(double) * (size_t)d);
    if (!cdf) return 2;
    double acc = 0.0;
    for (int32_t i = 0; i < d; ++i) { acc += pow((double)(i + 1), -g->zipf_a); cdf[i] = acc; }
  }
  int err = 0;
#pragma omp parallel
  {
    uint8_t* seen = (uint8_t*)calloc((size_t)d, 1);
    double* vtmp = (double*)malloc(sizeof(double) * (size_t)(d > 0 ? d : 1));
    if (!seen || !vtmp) {
#pragma omp atomic write
      err = 2;
    } else {
#pragma omp for schedule(dynamic, 256)
      for (int64_t i = 0; i < n; ++i) {
        rng_t r = row_rng(g, row0 + i);
        int32_t c = draw_count(g, &r);
        int64_t base = indptr[i];
        if (indptr[i + 1] - base != c) { err = 3; continue; }
        int32_t* out = indices + base;
        for (int32_t j = 0; j < c;) {
          int32_t f;
          if (g->feat_law == 0) {
            f = (int32_t)(unif(&r) * d);
          } else if (g->feat_law == 1) {
            double u = unif(&r) * cdf[d - 1];
            int32_t lo = 0, hi = d - 1; /* smallest i with cdf[i] > u */
            while (lo < hi) { int32_t mid = (lo + hi) >> 1; if (cdf[mid] > u) hi = mid; else lo = mid + 1; }
            f = lo;
          } else {
            int32_t band = (int32_t)(unif(&r) * g->n_bands);
            double centre = (2.0 * band + 1.0) * (double)d / (2.0 * g->n_bands);
            double x = centre + g->band_sigma * normal(&r);
            if (x < 0.0 || x >= (double)d) continue;
            f = (int32_t)floor(x);
          }
          if (f < 0 || f >= d || seen[f]) continue;
          seen[f] = 1;
          out[j++] = f;
        }
        for (int32_t j = 0; j < c; ++j) seen[out[j]] = 0;
        qsort(out, (size_t)c, sizeof(int32_t), cmp_i32);
        if (g->value_law == 1) {
          float* v = (float*)values + base;
          for (int32_t j = 0; j < c; ++j) v[j] = (float)exp(normal(&r));
        } else if (g->value_law == 2) {
          float* v = (float*)values + base;
          double ss = 0.0;
          for (int32_t j = 0; j < c; ++j) { vtmp[j] = exp(normal(&r)); ss += vtmp[j] * vtmp[j]; }
          double inv = ss > 0.0 ? 1.0 / sqrt(ss) : 0.0;
          for (int32_t j = 0; j < c; ++j) v[j] = (float)(vtmp[j] * inv);
        } else if (g->value_law == 3) {
          int8_t* v = (int8_t*)values + base;
          int32_t span = g->val_hi - g->val_lo + 1;
          for (int32_t j = 0; j < c; ++j) v[j] = (int8_t)(g->val_lo + (int32_t)(unif(&r) * span));
        }
      }
    }
    free(seen);
    free(vtmp);
  }
  free(cdf);
  return err;
}
