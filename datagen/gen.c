/*
 * datagen/gen.c — seeded synthetic sparse-vector generators.
 *
 * Test/bench infrastructure shared by BOTH the oracle (oracle/) and the CUDA
 * path (paper_2301_10622_b200/): it only draws random inputs and holds none
 * of Sinnamon's arithmetic (no sketching, decoding, scoring or selection).
 *
 * Every row r of stream s is drawn from its own counter-based generator
 * seeded by (seed, s, r), so any row can be regenerated independently, by any
 * thread, in any order, with identical results (used to regenerate sampled
 * documents of the 8.8 M-document config on the oracle side).
 *
 * Recipe:
 *   nnz:     fixed | uniform{a..b} | Poisson(a) clipped | round(LogNormal(a,b)) clipped
 *   coords:  uniform without replacement (Floyd) | Zipf(s) over ranks 1..n without
 *            replacement (successive sampling: draw with replacement, reject repeats),
 *            rank r -> coordinate r-1; sorted ascending in the output row
 *   values:  Normal(a,b) | LogNormal(a,b) | Laplace(a,b) | Uniform[a,b), cast to fp32,
 *            drawn in ascending-coordinate order
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int32_t n;         /* dimensionality */
  int32_t nnz_kind;  /* 0 fixed(a) 1 uniform{a..b} 2 poisson(a) 3 lognormal(mu=a, sigma=b) */
  double nnz_a, nnz_b;
  int32_t nnz_lo, nnz_hi; /* clip range (inclusive) */
  int32_t coord_kind;     /* 0 uniform w/o replacement, 1 zipf(zipf_s) w/o replacement */
  double zipf_s;
  int32_t val_kind;       /* 0 normal(a,b) 1 lognormal(a,b) 2 laplace(a,b) 3 uniform[a,b) */
  double val_a, val_b;
} gen_spec;

/* ---- counter-based RNG: splitmix64 stream seeded from (seed, stream, row) ---- */
typedef struct { uint64_t s; } rng_t;

static inline uint64_t sm_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static inline void rng_init(rng_t* r, uint64_t seed, uint64_t stream, uint64_t row) {
  uint64_t z = sm_mix(seed + 0x9E3779B97F4A7C15ull);
  z = sm_mix(z ^ (stream * 0xD1B54A32D192ED03ull));
  z = sm_mix(z ^ (row * 0x8CB92BA72F3D8DD7ull + 0x632BE59BD9B4E019ull));
  r->s = z;
}
static inline uint64_t rng_u64(rng_t* r) {
  r->s += 0x9E3779B97F4A7C15ull;
  return sm_mix(r->s);
}
/* uniform double in [0,1) with 53 random bits */
static inline double rng_unif(rng_t* r) { return (double)(rng_u64(r) >> 11) * (1.0 / 9007199254740992.0); }
/* uniform double in (0,1] */
static inline double rng_unif_pos(rng_t* r) { return ((double)(rng_u64(r) >> 11) + 1.0) * (1.0 / 9007199254740992.0); }
/* uniform integer in [0, bound) (Lemire multiply-shift, bias < 2^-32 for bound < 2^32) */
static inline uint32_t rng_below(rng_t* r, uint32_t bound) {
  return (uint32_t)(((__uint128_t)rng_u64(r) * (__uint128_t)bound) >> 64);
}
static inline double rng_normal(rng_t* r) {
  double u1 = rng_unif_pos(r), u2 = rng_unif(r);
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925 * u2);
}
static int32_t rng_poisson(rng_t* r, double lam) {
  /* inversion by sequential search; exact for lam up to ~700 (exp(-lam) > DBL_MIN) */
  double u = rng_unif(r), p = exp(-lam), F = p;
  int32_t k = 0;
  while (u > F && k < 100000) { k++; p *= lam / k; F += p; }
  return k;
}

static int32_t draw_nnz(const gen_spec* g, rng_t* r) {
  int64_t k;
  switch (g->nnz_kind) {
    case 0: k = (int64_t)g->nnz_a; break;
    case 1: k = (int64_t)g->nnz_a + rng_below(r, (uint32_t)((int64_t)g->nnz_b - (int64_t)g->nnz_a + 1)); break;
    case 2: k = rng_poisson(r, g->nnz_a); break;
    default: k = (int64_t)llround(exp(g->nnz_a + g->nnz_b * rng_normal(r))); break;
  }
  if (k < g->nnz_lo) k = g->nnz_lo;
  if (k > g->nnz_hi) k = g->nnz_hi;
  if (k > g->n) k = g->n;
  if (k < 0) k = 0;
  return (int32_t)k;
}

static float draw_val(const gen_spec* g, rng_t* r) {
  double v;
  switch (g->val_kind) {
    case 0: v = g->val_a + g->val_b * rng_normal(r); break;
    case 1: v = exp(g->val_a + g->val_b * rng_normal(r)); break;
    case 2: {
      double u = rng_unif(r) - 0.5; /* [-0.5, 0.5) */
      double a = fabs(u);
      if (a >= 0.5) a = 0.4999999999999999;
      v = g->val_a - g->val_b * (u < 0 ? -1.0 : 1.0) * log(1.0 - 2.0 * a);
      break;
    }
    default: v = g->val_a + (g->val_b - g->val_a) * rng_unif(r); break;
  }
  return (float)v;
}

static int cmp_i32(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

/* Fill one row: coords sorted ascending, then values. stamp: per-thread int32[n]. */
static void fill_row(const gen_spec* g, const double* zcdf, uint64_t seed, uint64_t stream, int64_t row,
                     int32_t nnz_expect, int32_t* idx, float* val, int32_t* stamp, int32_t tag) {
  rng_t r;
  rng_init(&r, seed, stream, (uint64_t)row);
  int32_t k = draw_nnz(g, &r);
  (void)nnz_expect;
  const int32_t n = g->n;
  if (g->coord_kind == 0) {
    /* Floyd's algorithm: k distinct values uniform over [0, n) */
    int32_t c = 0;
    for (int32_t j = n - k; j < n; j++) {
      int32_t t = (int32_t)rng_below(&r, (uint32_t)(j + 1));
      if (stamp[t] == tag) t = j;
      stamp[t] = tag;
      idx[c++] = t;
    }
  } else {
    /* successive sampling from Zipf(s) over ranks 1..n without replacement */
    int32_t c = 0;
    int64_t draws = 0, limit = 64LL * k + 100000;
    while (c < k && draws < limit) {
      double u = rng_unif(&r);
      /* smallest rank index t with zcdf[t] > u */
      int32_t lo = 0, hi = n - 1;
      while (lo < hi) {
        int32_t mid = lo + ((hi - lo) >> 1);
        if (zcdf[mid] > u) hi = mid; else lo = mid + 1;
      }
      draws++;
      if (stamp[lo] == tag) continue;
      stamp[lo] = tag;
      idx[c++] = lo;
    }
    for (int32_t t = 0; c < k && t < n; t++) /* pathological tail: deterministic top-up */
      if (stamp[t] != tag) { stamp[t] = tag; idx[c++] = t; }
  }
  qsort(idx, (size_t)k, sizeof(int32_t), cmp_i32);
  for (int32_t e = 0; e < k; e++) val[e] = draw_val(g, &r);
}

static double* make_zcdf(const gen_spec* g) {
  if (g->coord_kind != 1) return NULL;
  double* c = (double*)malloc(sizeof(double) * (size_t)g->n);
  double acc = 0.0;
  for (int32_t t = 0; t < g->n; t++) { acc += pow((double)(t + 1), -g->zipf_s); c[t] = acc; }
  for (int32_t t = 0; t < g->n; t++) c[t] /= acc;
  c[g->n - 1] = 1.0;
  return c;
}

/* nnz of rows [start, start+count) -> indptr[0..count] (indptr[0] = 0). Returns total nnz. */
int64_t gen_count(const gen_spec* g, uint64_t seed, uint64_t stream, int64_t start, int64_t count, int64_t* indptr) {
  indptr[0] = 0;
  for (int64_t r = 0; r < count; r++) {
    rng_t rr;
    rng_init(&rr, seed, stream, (uint64_t)(start + r));
    indptr[r + 1] = indptr[r] + draw_nnz(g, &rr);
  }
  return indptr[count];
}

typedef struct {
  const gen_spec* g; const double* zcdf; uint64_t seed, stream; int64_t start, r0, r1;
  const int64_t* indptr; int32_t* indices; float* values;
} fill_job;

static void* fill_worker(void* arg) {
  fill_job* J = (fill_job*)arg;
  int32_t* stamp = (int32_t*)malloc(sizeof(int32_t) * (size_t)J->g->n);
  for (int32_t t = 0; t < J->g->n; t++) stamp[t] = -1;
  int32_t tag = 0;
  for (int64_t r = J->r0; r < J->r1; r++) {
    int64_t o = J->indptr[r];
    fill_row(J->g, J->zcdf, J->seed, J->stream, J->start + r, (int32_t)(J->indptr[r + 1] - o),
             J->indices + o, J->values + o, stamp, tag);
    if (++tag == 0x7fffffff) { for (int32_t t = 0; t < J->g->n; t++) stamp[t] = -1; tag = 0; }
  }
  free(stamp);
  return NULL;
}

/* Fill rows [start, start+count) into indices/values using indptr from gen_count. */
int gen_fill(const gen_spec* g, uint64_t seed, uint64_t stream, int64_t start, int64_t count,
             const int64_t* indptr, int32_t* indices, float* values, int nthreads) {
  double* zcdf = make_zcdf(g);
  if (nthreads < 1) nthreads = 1;
  if (count < 4096) nthreads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
  fill_job* jobs = (fill_job*)malloc(sizeof(fill_job) * (size_t)nthreads);
  for (int t = 0; t < nthreads; t++) {
    jobs[t] = (fill_job){g, zcdf, seed, stream, start, count * t / nthreads, count * (t + 1) / nthreads,
                         indptr, indices, values};
    if (nthreads == 1) fill_worker(&jobs[t]);
    else pthread_create(&th[t], NULL, fill_worker, &jobs[t]);
  }
  if (nthreads > 1)
    for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
  free(th); free(jobs); free(zcdf);
  return 0;
}

/* n*h table of bucket ids, uniform over [0, m): out[j*h + o]. Row j uses RNG (seed, stream, j). */
void gen_table(int32_t n, int32_t h, int32_t m, uint64_t seed, uint64_t stream, int32_t* out) {
  for (int32_t j = 0; j < n; j++) {
    rng_t r;
    rng_init(&r, seed, stream, (uint64_t)j);
    for (int32_t o = 0; o < h; o++) out[(int64_t)j * h + o] = (int32_t)rng_below(&r, (uint32_t)m);
  }
}

/* count distinct values chosen uniformly without replacement from pool[0..npool) (partial Fisher-Yates). */
void gen_choose(const uint32_t* pool, int64_t npool, int64_t count, uint64_t seed, uint64_t stream, uint64_t row,
                uint32_t* out) {
  uint32_t* tmp = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(npool > 0 ? npool : 1));
  memcpy(tmp, pool, sizeof(uint32_t) * (size_t)npool);
  rng_t r;
  rng_init(&r, seed, stream, row);
  if (count > npool) count = npool;
  for (int64_t i = 0; i < count; i++) {
    int64_t j = i + (int64_t)(((__uint128_t)rng_u64(&r) * (__uint128_t)(uint64_t)(npool - i)) >> 64);
    uint32_t t = tmp[i]; tmp[i] = tmp[j]; tmp[j] = t;
    out[i] = tmp[i];
  }
  free(tmp);
}
