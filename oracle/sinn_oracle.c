/*
 * oracle/sinn_oracle.c — plain, slow, obviously-correct CPU oracle of Sinnamon
 * (Bruch, Nardini, Ingber, Liberty: "An Approximate Algorithm for Maximum Inner
 * Product Search over Streaming Sparse Vectors", arXiv 2301.10622).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or helper with the CUDA path (paper_2301_10622_b200/).
 *
 * Citations are PAPER.md lines ("P:N") and the algorithm they sit in.
 *   Alg. 5 Indexing   P:309-327 (sketch u = max, l = min over colliding coords)
 *   Sinnamon+         P:358     (upper sketch only, non-negative orthant)
 *   Alg. 6 Scoring    P:383-409 (walk I[j] for j in nz(q) sorted by |q_j| desc;
 *                                min over U rows if q_j > 0, max over L rows otherwise)
 *   Alg. 7 Ranking    P:415-435 (FindLargest k', exact re-rank, FindLargest k; k' >= k)
 *   Alg. 3 FindLargest P:232-252 (bounded min-heap, admit only if score > theta)
 *   Deletion          P:460-468 (remove i from every I[j]; sketch column left stale; id reusable)
 *   Exact MIPS        Eq. (2) / Alg. 2 P:212-256 (sum q_j x_j; unvisited docs score 0)
 * Readings where the paper is silent are DESIGN.md "Readings" R1..R17.
 * Arithmetic: sketches hold the inserted fp32 values exactly (max/min do not round);
 * every score is accumulated in fp64.  ORC_SKETCH_BF16 (the paper's
 * compressed store): every sketch cell is stored in bfloat16 with directed
 * rounding — U cells rounded up, L cells rounded down — so each decode still bounds x_j from
 * the correct side and Theorem 1 holds (reading R21).
 *
 * Parity pins (tests/test_oracle_*.py): O1 sandwich, O2 max/min exact, O3 brute-force
 * collision characterisation, O4 injective table => exact, O5 Theorem 1, O6 gap
 * identity, O7/O8 closed form vs Monte Carlo vs Table 1, O9 dense brute force,
 * O10 k' = |X| => exact top-k, O11 Sinnamon+ == Sinnamon on non-negative data,
 * O12 postings == recomputation from the raw store.  No function is "parity unpinned".
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { ORC_OK = 0, ORC_EINVAL = 1, ORC_ENOMEM = 2, ORC_EEXIST = 3, ORC_ENOTFOUND = 4 };
enum { ORC_UPPER_ONLY = 1u, ORC_SKETCH_BF16 = 2u };
#define ORC_NO_ID 0xFFFFFFFFu

typedef struct {
  int32_t n, m, h;
  uint32_t flags;
  int32_t* pi;        /* pi[j*h + o] = pi_o(j), the h random mappings [n] -> [m] */
  int64_t cap;        /* columns allocated in the sketch matrix */
  float* U;           /* U^T[i] = column i of the upper sketch, m cells: U[i*m + k] */
  float* L;           /* L^T[i]: lower sketch (absent under Sinnamon+) */
  uint8_t* live;      /* i in X */
  int32_t* raw_nnz;   /* vector storage S: raw x_i for Fetch */
  int32_t** raw_idx;
  float** raw_val;
  uint32_t** inv;     /* inverted index I[j]: sorted ids (ordered set) */
  int64_t* inv_len;
  int64_t* inv_cap;
} orc_index;

/* ------------------------------------------------------------------ bfloat16, directed rounding (R21) */
/* bfloat16 = the fp32 values whose low 16 bits are zero (same sign and exponent fields, 7
 * mantissa bits).  orc_bf16_up(x) is the smallest bfloat16 >= x; orc_bf16_down(x) the largest
 * bfloat16 <= x (= -orc_bf16_up(-x)).  Infinities are bfloat16 already; NaN never reaches here. */
float orc_bf16_up(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  if ((u & 0xFFFFu) == 0) return x;       /* representable */
  uint32_t t = u & 0xFFFF0000u;            /* truncation: toward zero */
  if (!(u & 0x80000000u)) t += 0x10000u;   /* x > 0: toward zero is down, so step one bf16 up
                                              (the largest finite steps to +inf) */
  float r;
  memcpy(&r, &t, 4);
  return r;
}
float orc_bf16_down(float x) { return -orc_bf16_up(-x); }

/* ------------------------------------------------------------------ create */
orc_index* orc_create(int32_t n, int32_t m, int32_t h, const int32_t* table, uint32_t flags) {
  if (n < 1 || m < 1 || h < 1) return NULL;
  for (int64_t t = 0; t < (int64_t)n * h; t++)
    if (table[t] < 0 || table[t] >= m) return NULL;
  orc_index* X = (orc_index*)calloc(1, sizeof(orc_index));
  X->n = n; X->m = m; X->h = h; X->flags = flags;
  X->pi = (int32_t*)malloc(sizeof(int32_t) * (size_t)n * (size_t)h);
  memcpy(X->pi, table, sizeof(int32_t) * (size_t)n * (size_t)h);
  X->inv = (uint32_t**)calloc((size_t)n, sizeof(uint32_t*));
  X->inv_len = (int64_t*)calloc((size_t)n, sizeof(int64_t));
  X->inv_cap = (int64_t*)calloc((size_t)n, sizeof(int64_t));
  return X;
}

void orc_destroy(orc_index* X) {
  if (!X) return;
  for (int64_t i = 0; i < X->cap; i++) { free(X->raw_idx[i]); free(X->raw_val[i]); }
  for (int32_t j = 0; j < X->n; j++) free(X->inv[j]);
  free(X->inv); free(X->inv_len); free(X->inv_cap);
  free(X->U); free(X->L); free(X->live); free(X->raw_nnz); free(X->raw_idx); free(X->raw_val);
  free(X->pi); free(X);
}

static void grow(orc_index* X, int64_t need) {
  if (need <= X->cap) return;
  int64_t c = X->cap ? X->cap : 1024;
  while (c < need) c *= 2;
  int64_t m = X->m;
  X->U = (float*)realloc(X->U, sizeof(float) * (size_t)(c * m));
  if (!(X->flags & ORC_UPPER_ONLY)) X->L = (float*)realloc(X->L, sizeof(float) * (size_t)(c * m));
  X->live = (uint8_t*)realloc(X->live, (size_t)c);
  X->raw_nnz = (int32_t*)realloc(X->raw_nnz, sizeof(int32_t) * (size_t)c);
  X->raw_idx = (int32_t**)realloc(X->raw_idx, sizeof(int32_t*) * (size_t)c);
  X->raw_val = (float**)realloc(X->raw_val, sizeof(float*) * (size_t)c);
  for (int64_t i = X->cap; i < c; i++) {
    X->live[i] = 0; X->raw_nnz[i] = 0; X->raw_idx[i] = NULL; X->raw_val[i] = NULL;
    for (int64_t k = 0; k < m; k++) {
      X->U[i * m + k] = -INFINITY;
      if (X->L) X->L[i * m + k] = INFINITY;
    }
  }
  X->cap = c;
}

/* ordered-set insert of id into I[j] (binary search + shift) */
static void inv_insert(orc_index* X, int32_t j, uint32_t id) {
  if (X->inv_len[j] == X->inv_cap[j]) {
    X->inv_cap[j] = X->inv_cap[j] ? 2 * X->inv_cap[j] : 8;
    X->inv[j] = (uint32_t*)realloc(X->inv[j], sizeof(uint32_t) * (size_t)X->inv_cap[j]);
  }
  uint32_t* a = X->inv[j];
  int64_t lo = 0, hi = X->inv_len[j];
  while (lo < hi) { int64_t mid = (lo + hi) / 2; if (a[mid] < id) lo = mid + 1; else hi = mid; }
  memmove(a + lo + 1, a + lo, sizeof(uint32_t) * (size_t)(X->inv_len[j] - lo));
  a[lo] = id;
  X->inv_len[j]++;
}

static void inv_remove(orc_index* X, int32_t j, uint32_t id) {
  uint32_t* a = X->inv[j];
  int64_t lo = 0, hi = X->inv_len[j];
  while (lo < hi) { int64_t mid = (lo + hi) / 2; if (a[mid] < id) lo = mid + 1; else hi = mid; }
  if (lo < X->inv_len[j] && a[lo] == id) {
    memmove(a + lo, a + lo + 1, sizeof(uint32_t) * (size_t)(X->inv_len[j] - lo - 1));
    X->inv_len[j]--;
  }
}

static int cmp_u32(const void* a, const void* b) {
  uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return (x > y) - (x < y);
}

/* ------------------------------------------------------------------ insert (Alg. 5) */
/* Validation is all-or-nothing (R18): a rejected batch changes nothing. */
int orc_insert(orc_index* X, int64_t nrows, const int64_t* indptr, const int32_t* indices, const float* values,
               const uint32_t* ids) {
  if (nrows < 0) return ORC_EINVAL;
  if (nrows == 0) return ORC_OK;
  for (int64_t r = 0; r < nrows; r++) {
    if (indptr[r + 1] < indptr[r]) return ORC_EINVAL;
    if (ids[r] == ORC_NO_ID) return ORC_EINVAL;
    for (int64_t e = indptr[r]; e < indptr[r + 1]; e++) {
      if (indices[e] < 0 || indices[e] >= X->n) return ORC_EINVAL;
      if (e > indptr[r] && indices[e] <= indices[e - 1]) return ORC_EINVAL;
      if (!isfinite(values[e])) return ORC_EINVAL;
      if ((X->flags & ORC_UPPER_ONLY) && values[e] < 0.0f) return ORC_EINVAL;
    }
  }
  uint32_t* sorted = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)nrows);
  memcpy(sorted, ids, sizeof(uint32_t) * (size_t)nrows);
  qsort(sorted, (size_t)nrows, sizeof(uint32_t), cmp_u32);
  for (int64_t r = 1; r < nrows; r++)
    if (sorted[r] == sorted[r - 1]) { free(sorted); return ORC_EINVAL; }
  free(sorted);
  for (int64_t r = 0; r < nrows; r++)
    if ((int64_t)ids[r] < X->cap && X->live[ids[r]]) return ORC_EEXIST;

  for (int64_t r = 0; r < nrows; r++) {
    const uint32_t i = ids[r];
    grow(X, (int64_t)i + 1);
    const int64_t b = indptr[r], nnz = indptr[r + 1] - indptr[r];
    /* line 1: nz(x_i) — the active (stored) coordinates (R4: a stored 0 is active) */
    /* line 2: I[j].Insert(i) for all j in nz(x_i) */
    for (int64_t e = 0; e < nnz; e++) inv_insert(X, indices[b + e], i);
    /* lines 3-7: u[k] = max, l[k] = min over {j in nz(x_i) : exists o, pi_o(j) = k};
       an empty set leaves the identity element (-inf for max, +inf for min; R1). */
    const int64_t m = X->m;
    float* u = X->U + (int64_t)i * m;
    float* l = X->L ? X->L + (int64_t)i * m : NULL;
    for (int64_t k = 0; k < m; k++) {
      u[k] = -INFINITY;
      if (l) l[k] = INFINITY;
    }
    for (int64_t e = 0; e < nnz; e++) {
      const int32_t j = indices[b + e];
      float x = values[b + e];
      if (x == 0.0f) x = 0.0f; /* R19: -0.0 is stored as +0.0 (equal reals) */
      for (int32_t o = 0; o < X->h; o++) {
        const int32_t k = X->pi[(int64_t)j * X->h + o];
        if (x > u[k]) u[k] = x;
        if (l && x < l[k]) l[k] = x;
      }
    }
    /* F3 (R21): the stored cell is the exact max (min) rounded up (down) to bfloat16 */
    if (X->flags & ORC_SKETCH_BF16)
      for (int64_t k = 0; k < m; k++) {
        u[k] = orc_bf16_up(u[k]);
        if (l) l[k] = orc_bf16_down(l[k]);
      }
    /* the raw vector goes to the vector storage S */
    free(X->raw_idx[i]); free(X->raw_val[i]);
    X->raw_nnz[i] = (int32_t)nnz;
    X->raw_idx[i] = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nnz > 0 ? nnz : 1));
    X->raw_val[i] = (float*)malloc(sizeof(float) * (size_t)(nnz > 0 ? nnz : 1));
    for (int64_t e = 0; e < nnz; e++) {
      X->raw_idx[i][e] = indices[b + e];
      X->raw_val[i][e] = values[b + e] == 0.0f ? 0.0f : values[b + e];
    }
    X->live[i] = 1;
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------ delete */
int orc_delete(orc_index* X, int64_t count, const uint32_t* ids) {
  if (count < 0) return ORC_EINVAL;
  uint32_t* sorted = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(count > 0 ? count : 1));
  memcpy(sorted, ids, sizeof(uint32_t) * (size_t)count);
  qsort(sorted, (size_t)count, sizeof(uint32_t), cmp_u32);
  for (int64_t r = 1; r < count; r++)
    if (sorted[r] == sorted[r - 1]) { free(sorted); return ORC_EINVAL; }
  free(sorted);
  for (int64_t r = 0; r < count; r++)
    if ((int64_t)ids[r] >= X->cap || !X->live[ids[r]]) return ORC_ENOTFOUND;
  for (int64_t r = 0; r < count; r++) {
    const uint32_t i = ids[r];
    /* remove every instance of i from the inverted lists; the sketch column is NOT cleaned */
    for (int32_t e = 0; e < X->raw_nnz[i]; e++) inv_remove(X, X->raw_idx[i][e], i);
    /* ... and i joins the set of available identifiers (the caller recycles it) */
    X->live[i] = 0;
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------ decode */
/* least upper bound (q_j > 0) or greatest lower bound (q_j < 0) of x_i[j] from the sketch.
   Under Sinnamon+ the lower bound of a non-negative value is 0 (R6). */
static double decode(const orc_index* X, uint32_t i, int32_t j, int positive) {
  const int64_t m = X->m;
  if (positive) {
    float e = INFINITY;
    for (int32_t o = 0; o < X->h; o++) {
      float c = X->U[(int64_t)i * m + X->pi[(int64_t)j * X->h + o]];
      if (c < e) e = c;
    }
    return (double)e;
  }
  if (X->flags & ORC_UPPER_ONLY) return 0.0;
  float e = -INFINITY;
  for (int32_t o = 0; o < X->h; o++) {
    float c = X->L[(int64_t)i * m + X->pi[(int64_t)j * X->h + o]];
    if (c > e) e = c;
  }
  return (double)e;
}

float orc_decode(const orc_index* X, uint32_t i, int32_t j, int positive) { return (float)decode(X, i, j, positive); }

/* ------------------------------------------------------------------ FindLargest (Alg. 3) */
/* Total order of FindLargest's output: score descending, then id ascending (R10: strict
   "> theta" admission while scanning ids in ascending order keeps the earlier id on ties).
   "worse(a, b)" = a ranks below b. */
typedef struct { double s; uint32_t id; } item;
static int worse(item a, item b) { return a.s < b.s || (a.s == b.s && a.id > b.id); }

static void sift_down(item* hp, int64_t n, int64_t p) {
  for (;;) {
    int64_t c = 2 * p + 1, w = p;
    if (c < n && worse(hp[c], hp[w])) w = c;
    if (c + 1 < n && worse(hp[c + 1], hp[w])) w = c + 1;
    if (w == p) return;
    item t = hp[p]; hp[p] = hp[w]; hp[w] = t; p = w;
  }
}
static void sift_up(item* hp, int64_t p) {
  while (p > 0) {
    int64_t par = (p - 1) / 2;
    if (!worse(hp[p], hp[par])) return;
    item t = hp[p]; hp[p] = hp[par]; hp[par] = t; p = par;
  }
}
static int cmp_rank(const void* a, const void* b) {
  item x = *(const item*)a, y = *(const item*)b;
  if (worse(x, y)) return 1;
  if (worse(y, x)) return -1;
  return 0;
}
/* heap of size k; theta = worst in heap once full; admit only if strictly better.
   Returns the number selected; out is sorted best-first. */
static int64_t find_largest(const item* cand, int64_t ncand, int64_t k, item* out) {
  int64_t sz = 0;
  for (int64_t t = 0; t < ncand; t++) {
    if (sz < k) { out[sz] = cand[t]; sift_up(out, sz); sz++; }
    else if (k > 0 && worse(out[0], cand[t])) { out[0] = cand[t]; sift_down(out, sz, 0); }
  }
  qsort(out, (size_t)sz, sizeof(item), cmp_rank);
  return sz;
}

int64_t orc_find_largest(const double* scores, const uint32_t* ids, int64_t n, int64_t k, uint32_t* out_ids,
                         double* out_scores) {
  item* c = (item*)malloc(sizeof(item) * (size_t)(n > 0 ? n : 1));
  item* o = (item*)malloc(sizeof(item) * (size_t)(k > 0 ? k : 1));
  for (int64_t t = 0; t < n; t++) { c[t].s = scores[t]; c[t].id = ids[t]; }
  int64_t r = find_largest(c, n, k, o);
  for (int64_t t = 0; t < r; t++) { out_ids[t] = o[t].id; out_scores[t] = o[t].s; }
  free(c); free(o);
  return r;
}

/* ------------------------------------------------------------------ scoring (Alg. 6) */
typedef struct { int32_t j; double q; } qterm;
static int cmp_qterm(const void* a, const void* b) {
  qterm x = *(const qterm*)a, y = *(const qterm*)b;
  double ax = fabs(x.q), ay = fabs(y.q);
  if (ax > ay) return -1;
  if (ax < ay) return 1;
  return (x.j > y.j) - (x.j < y.j);
}

/* scores[i] for every column i < cap (vacant columns get -inf: never selected, R9);
   mass[i] = sum |q_j * e_ij| (tolerance scale, R7) if mass != NULL.
   max_terms > 0: the anytime budget of Alg. 6 read as a number of query terms
   (R20): only the first max_terms terms of the |q_j|-descending order are processed. */
static void score_query(const orc_index* X, int64_t qnnz, const int32_t* qidx, const float* qval, double* scores,
                        double* mass, int32_t max_terms) {
  /* line 1: nz(q) = {j : q[j] != 0} */
  qterm* t = (qterm*)malloc(sizeof(qterm) * (size_t)(qnnz > 0 ? qnnz : 1));
  int64_t nt = 0;
  for (int64_t e = 0; e < qnnz; e++)
    if (qval[e] != 0.0f) { t[nt].j = qidx[e]; t[nt].q = (double)qval[e]; nt++; }
  /* line 2: sort by |q[j]| descending (ties: ascending j, R14) — fixes the fp64 summation order */
  qsort(t, (size_t)nt, sizeof(qterm), cmp_qterm);
  /* line 3: scores[i] = 0 for all i in X */
  for (int64_t i = 0; i < X->cap; i++) {
    scores[i] = X->live[i] ? 0.0 : -INFINITY;
    if (mass) mass[i] = 0.0;
  }
  /* lines 4-13; line 12: stop once the budget is spent */
  const int64_t nproc = (max_terms > 0 && max_terms < nt) ? max_terms : nt;
  for (int64_t a = 0; a < nproc; a++) {
    const int32_t j = t[a].j;
    const double q = t[a].q;
    for (int64_t p = 0; p < X->inv_len[j]; p++) {
      const uint32_t i = X->inv[j][p];
      const double s = q * decode(X, i, j, q > 0);
      scores[i] += s;
      if (mass) mass[i] += fabs(s);
    }
  }
  free(t);
}

int orc_score(const orc_index* X, int64_t qnnz, const int32_t* qidx, const float* qval, double* scores, double* mass) {
  score_query(X, qnnz, qidx, qval, scores, mass, 0);
  return ORC_OK;
}

int orc_score_budget(const orc_index* X, int64_t qnnz, const int32_t* qidx, const float* qval, int32_t max_terms,
                     double* scores, double* mass) {
  score_query(X, qnnz, qidx, qval, scores, mass, max_terms);
  return ORC_OK;
}

/* exact <q, x_i> from the vector storage: sum over nz(q) ∩ nz(x_i) of q_j x_ij (fp64) */
static double exact_dot(const orc_index* X, uint32_t i, int64_t qnnz, const int32_t* qidx, const float* qval) {
  double s = 0.0;
  int64_t a = 0, b = 0;
  const int32_t* di = X->raw_idx[i];
  const float* dv = X->raw_val[i];
  while (a < qnnz && b < X->raw_nnz[i]) {
    if (qidx[a] < di[b]) a++;
    else if (qidx[a] > di[b]) b++;
    else { s += (double)qval[a] * (double)dv[b]; a++; b++; }
  }
  return s;
}

double orc_exact_dot(const orc_index* X, uint32_t i, int64_t qnnz, const int32_t* qidx, const float* qval) {
  return exact_dot(X, i, qnnz, qidx, qval);
}

int64_t orc_cap(const orc_index* X) { return X->cap; }
int64_t orc_live_count(const orc_index* X) {
  int64_t c = 0;
  for (int64_t i = 0; i < X->cap; i++) c += X->live[i];
  return c;
}

/* ------------------------------------------------------------------ search (Alg. 6 + Alg. 7) */
typedef struct {
  const orc_index* X;
  const int64_t* qptr; const int32_t* qidx; const float* qval;
  int64_t k, kp; int rerank, exact;
  int32_t max_terms;                           /* anytime budget (terms), 0 = T infinity */
  const uint32_t* allow; int64_t allow_words;  /* constrained search (Eq. 3): column mask, NULL = all */
  uint32_t* out_ids; double* out_scores;       /* nq*k */
  uint32_t* cand_ids; double* cand_scores; double* cand_mass; /* nq*kp (optional) */
  int64_t q0, q1;
} search_job;

static void search_one(const search_job* J, int64_t qi, double* scores, double* mass, item* all, item* V, item* R) {
  const orc_index* X = J->X;
  const int64_t b = J->qptr[qi], qn = J->qptr[qi + 1] - J->qptr[qi];
  const int32_t* qidx = J->qidx + b;
  const float* qval = J->qval + b;
  int64_t nall = 0;
  if (J->exact) {
    /* Exact MIPS (Eq. 2; unvisited documents score 0) */
    for (int64_t i = 0; i < X->cap; i++)
      if (X->live[i]) { all[nall].s = exact_dot(X, (uint32_t)i, qn, qidx, qval); all[nall].id = (uint32_t)i; nall++; }
    int64_t r = find_largest(all, nall, J->k, R);
    for (int64_t t = 0; t < J->k; t++) {
      J->out_ids[qi * J->k + t] = t < r ? R[t].id : ORC_NO_ID;
      J->out_scores[qi * J->k + t] = t < r ? R[t].s : -INFINITY;
    }
    return;
  }
  score_query(X, qn, qidx, qval, scores, mass, J->max_terms);
  for (int64_t i = 0; i < X->cap; i++) {
    /* Eq. 3: a column whose document fails the constraints is masked out of the
       solution set, exactly as a vacant column (R9) */
    const int ok = !J->allow || (i < 32 * J->allow_words && ((J->allow[i >> 5] >> (i & 31)) & 1u));
    if (X->live[i] && ok) { all[nall].s = scores[i]; all[nall].id = (uint32_t)i; nall++; }
  }
  /* Alg. 7 line 1: V = FindLargest(scores, k') */
  int64_t nv = find_largest(all, nall, J->kp, V);
  if (J->cand_ids)
    for (int64_t t = 0; t < J->kp; t++) {
      J->cand_ids[qi * J->kp + t] = t < nv ? V[t].id : ORC_NO_ID;
      J->cand_scores[qi * J->kp + t] = t < nv ? V[t].s : -INFINITY;
      if (J->cand_mass) J->cand_mass[qi * J->kp + t] = t < nv ? mass[V[t].id] : 0.0;
    }
  int64_t nr;
  if (J->rerank) {
    /* lines 2-4: s_v = <q, S.Fetch(v)> */
    for (int64_t t = 0; t < nv; t++) V[t].s = exact_dot(X, V[t].id, qn, qidx, qval);
    /* line 5: FindLargest({s_v}, k) */
    nr = find_largest(V, nv, J->k, R);
  } else {
    nr = nv < J->k ? nv : J->k;
    memcpy(R, V, sizeof(item) * (size_t)nr);
  }
  for (int64_t t = 0; t < J->k; t++) {
    J->out_ids[qi * J->k + t] = t < nr ? R[t].id : ORC_NO_ID;
    J->out_scores[qi * J->k + t] = t < nr ? R[t].s : -INFINITY;
  }
}

static void* search_worker(void* arg) {
  search_job* J = (search_job*)arg;
  const int64_t cap = J->X->cap > 0 ? J->X->cap : 1;
  double* scores = (double*)malloc(sizeof(double) * (size_t)cap);
  double* mass = (double*)malloc(sizeof(double) * (size_t)cap);
  item* all = (item*)malloc(sizeof(item) * (size_t)cap);
  item* V = (item*)malloc(sizeof(item) * (size_t)(J->kp > 0 ? J->kp : 1));
  item* R = (item*)malloc(sizeof(item) * (size_t)(J->k > 0 ? J->k : 1));
  for (int64_t qi = J->q0; qi < J->q1; qi++) search_one(J, qi, scores, mass, all, V, R);
  free(scores); free(mass); free(all); free(V); free(R);
  return NULL;
}

static int validate_queries(const orc_index* X, int64_t nq, const int64_t* qptr, const int32_t* qidx,
                            const float* qval) {
  for (int64_t r = 0; r < nq; r++) {
    if (qptr[r + 1] < qptr[r]) return ORC_EINVAL;
    for (int64_t e = qptr[r]; e < qptr[r + 1]; e++) {
      if (qidx[e] < 0 || qidx[e] >= X->n) return ORC_EINVAL;
      if (e > qptr[r] && qidx[e] <= qidx[e - 1]) return ORC_EINVAL;
      if (!isfinite(qval[e])) return ORC_EINVAL;
    }
  }
  return ORC_OK;
}

static int run_jobs(search_job* proto, int64_t nq, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > nq) nthreads = (int)(nq > 0 ? nq : 1);
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
  search_job* jobs = (search_job*)malloc(sizeof(search_job) * (size_t)nthreads);
  for (int t = 0; t < nthreads; t++) {
    jobs[t] = *proto;
    jobs[t].q0 = nq * t / nthreads;
    jobs[t].q1 = nq * (t + 1) / nthreads;
    if (nthreads == 1) search_worker(&jobs[t]);
    else pthread_create(&th[t], NULL, search_worker, &jobs[t]);
  }
  if (nthreads > 1)
    for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
  free(th); free(jobs);
  return ORC_OK;
}

/* Search a batch: out (ids, scores) are nq*k, best first, padded (ORC_NO_ID, -inf).
   cand_* (nq*kprime, optional): the stage-1 set V with approximate scores and masses. */
int orc_search(const orc_index* X, int64_t nq, const int64_t* qptr, const int32_t* qidx, const float* qval, int32_t k,
               int32_t kprime, int32_t rerank, uint32_t* out_ids, double* out_scores, uint32_t* cand_ids,
               double* cand_scores, double* cand_mass, int nthreads) {
  if (nq < 0 || k < 1 || kprime < k) return ORC_EINVAL; /* k' >= k */
  if (validate_queries(X, nq, qptr, qidx, qval)) return ORC_EINVAL;
  search_job J = {X, qptr, qidx, qval, k, kprime, rerank, 0, 0, NULL, 0, out_ids, out_scores, cand_ids, cand_scores,
                  cand_mass, 0, 0};
  return run_jobs(&J, nq, nthreads);
}

/* As orc_search with the anytime budget: stage 1 scores only each query's first max_terms terms by
   descending |q_j| (Alg. 6 with budget T); the re-rank uses the whole query (Alg. 7). */
int orc_search_budget(const orc_index* X, int64_t nq, const int64_t* qptr, const int32_t* qidx, const float* qval,
                      int32_t k, int32_t kprime, int32_t rerank, int32_t max_terms, uint32_t* out_ids,
                      double* out_scores, uint32_t* cand_ids, double* cand_scores, double* cand_mass, int nthreads) {
  if (nq < 0 || k < 1 || kprime < k || max_terms < 0) return ORC_EINVAL;
  if (validate_queries(X, nq, qptr, qidx, qval)) return ORC_EINVAL;
  search_job J = {X, qptr, qidx, qval, k, kprime, rerank, 0, max_terms, NULL, 0, out_ids, out_scores, cand_ids,
                  cand_scores, cand_mass, 0, 0};
  return run_jobs(&J, nq, nthreads);
}

/* Constrained search (Eq. 3): as orc_search_budget, with only the documents whose bit is
   set in allow[0 .. allow_words) (bit i of word i/32) in the solution set. */
int orc_search_filtered(const orc_index* X, int64_t nq, const int64_t* qptr, const int32_t* qidx, const float* qval,
                        int32_t k, int32_t kprime, int32_t rerank, int32_t max_terms, const uint32_t* allow,
                        int64_t allow_words, uint32_t* out_ids, double* out_scores, int nthreads) {
  if (nq < 0 || k < 1 || kprime < k || max_terms < 0 || allow_words < 0) return ORC_EINVAL;
  if (validate_queries(X, nq, qptr, qidx, qval)) return ORC_EINVAL;
  search_job J = {X, qptr, qidx, qval, k, kprime, rerank, 0, max_terms, allow, allow_words, out_ids, out_scores, NULL,
                  NULL, NULL, 0, 0};
  return run_jobs(&J, nq, nthreads);
}

/* Exact top-k over the live collection (ground truth for recall@k). */
int orc_exact(const orc_index* X, int64_t nq, const int64_t* qptr, const int32_t* qidx, const float* qval, int32_t k,
              uint32_t* out_ids, double* out_scores, int nthreads) {
  if (nq < 0 || k < 1) return ORC_EINVAL;
  if (validate_queries(X, nq, qptr, qidx, qval)) return ORC_EINVAL;
  search_job J = {X, qptr, qidx, qval, k, k, 0, 1, 0, NULL, 0, out_ids, out_scores, NULL, NULL, NULL, 0, 0};
  return run_jobs(&J, nq, nthreads);
}

/* ------------------------------------------------------------------ exports for parity */
int orc_export_sketch(const orc_index* X, int64_t count, const uint32_t* ids, float* U, float* L) {
  for (int64_t r = 0; r < count; r++) {
    if ((int64_t)ids[r] >= X->cap) return ORC_ENOTFOUND;
    memcpy(U + r * X->m, X->U + (int64_t)ids[r] * X->m, sizeof(float) * (size_t)X->m);
    if (L && X->L) memcpy(L + r * X->m, X->L + (int64_t)ids[r] * X->m, sizeof(float) * (size_t)X->m);
  }
  return ORC_OK;
}

int64_t orc_postings_len(const orc_index* X, int32_t j) { return (j >= 0 && j < X->n) ? X->inv_len[j] : -1; }
int orc_export_postings(const orc_index* X, int32_t j, uint32_t* out) {
  if (j < 0 || j >= X->n) return ORC_EINVAL;
  memcpy(out, X->inv[j], sizeof(uint32_t) * (size_t)X->inv_len[j]);
  return ORC_OK;
}
int orc_is_live(const orc_index* X, uint32_t i) { return (int64_t)i < X->cap && X->live[i]; }
int32_t orc_raw_nnz(const orc_index* X, uint32_t i) { return (int64_t)i < X->cap ? X->raw_nnz[i] : -1; }
int orc_raw_row(const orc_index* X, uint32_t i, int32_t* idx, float* val) {
  if ((int64_t)i >= X->cap) return ORC_ENOTFOUND;
  memcpy(idx, X->raw_idx[i], sizeof(int32_t) * (size_t)X->raw_nnz[i]);
  memcpy(val, X->raw_val[i], sizeof(float) * (size_t)X->raw_nnz[i]);
  return ORC_OK;
}

/* ------------------------------------------------------------------ stand-alone sketch (Alg. 5 lines 3-7) */
/* Sketch of one vector without an index (used by pins O1-O4, O7). */
void orc_sketch_row(int32_t m, int32_t h, const int32_t* pi, int64_t nnz, const int32_t* idx, const float* val,
                    float* u, float* l) {
  for (int32_t k = 0; k < m; k++) { u[k] = -INFINITY; if (l) l[k] = INFINITY; }
  for (int64_t e = 0; e < nnz; e++) {
    float x = val[e] == 0.0f ? 0.0f : val[e];
    for (int32_t o = 0; o < h; o++) {
      int32_t k = pi[(int64_t)idx[e] * h + o];
      if (x > u[k]) u[k] = x;
      if (l && x < l[k]) l[k] = x;
    }
  }
}
