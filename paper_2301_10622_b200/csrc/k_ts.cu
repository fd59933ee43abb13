// k_ts.cu — the tile-owned scoring kernel k_ts_score for head-heavy batches (Zipf configs 3 and 5):
// S1 (Alg. 6 walk + decode + accumulate) and the S2 threshold (Alg. 3 / Alg. 7
// line 1) for a pass of up to 1,024 queries, plus the batch preparation it
// needs (term classes, head-term query rows).
//
// Why a second kernel.  In configs 3 and 5 every query touches every document
// and a few hundred terms carry ~90 % of Alg. 6's (document, query) updates: config 5 walks 34.8 G
// updates per batch, config 3 120 G.  A per-document walk that re-reads each term's (query, q_j)
// pairs from L2 for every document holding the term (k_doc_score) moves ~8 B of L2 traffic per
// update; here a CTA owns a tile of 32 documents and every term present in the tile is handled ONCE
// for all of the tile's documents that hold it, by the cheapest of three forms:
//
//   head terms   (coverage df/N x nq/B >= tau, at most H per batch) — a dense register-tiled FP32
//                product  S[32 x 1024] += E[32 x H] . Q[H x 1024]  with E the decoded estimates
//                (0 where the document lacks the term) and Q the batch's q_j (0 where the query lacks
//                it); two-sided indexes split Q into q+ = max(q, 0) and q- = min(q, 0), which pick the
//                upper and lower estimate (Alg. 6 lines 7-10) with no select per update.  FFMA only
//                (BASELINE.json: no tensor cores; fp32 parity).
//   wide terms   (>= W_MIN queries of the pass) — term-major: the term's pairs are loaded once per
//                tile (lane = pair, bank-major order) and each document of the tile holding the term
//                adds q_j * e into its shared-memory score row: the update is LDS + FFMA + STS, the
//                shared-memory bound of 16 updates / clock / SM (tools/mb measurement).
//   other terms  — inside the per-document decode pass: terms with <= 8 queries lane = entry (tag
//                arrays serialise lanes that meet the same query), 9..W_MIN-1 queries warp-wide.
//
// Per 32-document tile (one index tile, entries (j << 5) | d grouped by document), 1,024 threads:
//   A  lane = entry over the tile: a byte per (wide term, document) present
//   .  masks of the wide terms, their slots in the tile's estimate list (block scan)
//   B  warp = document: decode every batch-term entry from the staged sketch column (min over the
//      h upper cells / max over the h lower cells, Alg. 6 lines 7-10): head -> E, wide -> its slot,
//      others -> added into S now
//   C  warps take wide terms from the tile's list (dynamic): term-major RMW into S; then each warp
//      runs its block of the dense head product in registers
//   D  every cell: S + head product, compared with theta_q (EMIT: a candidate; HIST: the sample
//      histogram); S reset.  The next tile's sketch streams into the staging buffer from B on.
// Scores never touch HBM.  Untouched documents score exactly 0 (R8).
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>

#include "sinn_device.cuh"
#include "sinn_internal.cuh"

namespace sinn {

namespace {

constexpr uint32_t kFullT = 0xffffffffu;
constexpr int kTD = 32;            // documents per tile (one index tile)
constexpr int kTQ = 1024;          // queries per pass
constexpr int kNWMax = 1024;       // wide terms per pass (batch-local ids)
constexpr int kTags = 128;         // per-warp conflict tags (query & 127)
constexpr int kHCand = 4096;       // head candidates considered per pass
constexpr int kTsHMax = 16;        // head terms per pass (upper bound of every instantiation)
constexpr int kThetaShiftT = 19;   // the sample histogram of k_tile.cu (k_theta)
constexpr int kThetaBinsT = 1 << (32 - kThetaShiftT);
constexpr uint32_t kClsShift = 30;
enum : uint32_t { kClsAbsent = 0, kClsSparse = 1, kClsWide = 2, kClsHead = 3 };

// ---------------------------------------------------------------- batch preparation
// coverage of term j = df[j]/live x (queries of the pass holding j)/nq: the expected fraction of
// (document, query) pairs it updates; candidates >= tau, best first (ties by term id)
__global__ void k_head_cand(const uint32_t* __restrict__ qoff, const int32_t* __restrict__ df, int32_t n,
                            float inv_live, float inv_nq, float tau, unsigned long long* __restrict__ cand,
                            uint32_t* __restrict__ ncand) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t qc = qoff[j + 1] - qoff[j];
    if (qc == 0) continue;
    const float cover = (float)df[j] * inv_live * ((float)qc * inv_nq);
    if (cover >= tau) {
      const uint32_t pos = atomicAdd(ncand, 1u);
      if (pos < (uint32_t)kHCand)
        cand[pos] = ((unsigned long long)__float_as_uint(cover) << 32) | (unsigned long long)(~(uint32_t)j);
    }
  }
}

// one block: the hmax best candidates -> head list hj[], the dense query rows Qh[hh][q] (q_j, 0 where
// the query lacks j), and the term's mark in the directory of the scoring kernel in use: dir (the
// 32-byte sector of k_doc_score: no sparse pairs, head mark) or tdir (k_ts_score: class head)
__global__ void __launch_bounds__(1024) k_head_pick(const unsigned long long* __restrict__ cand,
                                                    const uint32_t* __restrict__ ncand,
                                                    const uint32_t* __restrict__ qoff, const uint2* __restrict__ pairs,
                                                    uint4* __restrict__ dir, uint2* __restrict__ tdir,
                                                    float* __restrict__ Qh, uint32_t* __restrict__ head_cnt, int hmax,
                                                    int qrow) {
  __shared__ unsigned long long sb[kHCand];
  __shared__ uint32_t hj[kTsHMax];
  const uint32_t cnt = min(*ncand, (uint32_t)kHCand);
  int N = 1;
  while (N < (int)cnt) N <<= 1;
  for (int t = threadIdx.x; t < N; t += blockDim.x) sb[t] = t < (int)cnt ? cand[t] : 0ull;
  for (int k = 2; k <= N; k <<= 1)
    for (int jj = k >> 1; jj > 0; jj >>= 1) {
      __syncthreads();
      for (int i = threadIdx.x; i < N; i += blockDim.x) {
        const int l = i ^ jj;
        if (l > i) {
          const unsigned long long a = sb[i], b = sb[l];
          if (((i & k) == 0) ? (a < b) : (a > b)) {
            sb[i] = b;
            sb[l] = a;
          }
        }
      }
    }
  __syncthreads();
  const int hc = (int)min(cnt, (uint32_t)min(hmax, kTsHMax));
  if (threadIdx.x < (unsigned)hc) hj[threadIdx.x] = ~(uint32_t)(sb[threadIdx.x] & 0xffffffffu);
  for (int t = threadIdx.x; t < hmax * qrow; t += blockDim.x) Qh[t] = 0.0f;
  __syncthreads();
  for (int hh = 0; hh < hc; hh++) {
    const uint32_t j = hj[hh];
    const uint32_t b = qoff[j], e = qoff[j + 1];
    for (uint32_t r = b + threadIdx.x; r < e; r += blockDim.x) {
      const uint2 pr = pairs[r];
      Qh[hh * qrow + pr.x] = __uint_as_float(pr.y);
    }
  }
  if (threadIdx.x < (unsigned)hc) {
    const uint32_t j = hj[threadIdx.x];
    if (dir) {
      uint4 a = dir[2 * (int64_t)j];
      a.y = (a.y & 0xc0000000u) | a.x;  // no sparse pairs: the term is in the dense product
      dir[2 * (int64_t)j] = a;
      uint4 b = dir[2 * (int64_t)j + 1];
      b.x = 0x80000000u | threadIdx.x;  // k_doc_score's head mark (kHeadMarkD) | hh
      dir[2 * (int64_t)j + 1] = b;
    }
    if (tdir) {
      uint2 a = tdir[j];
      a.x = (kClsHead << kClsShift) | threadIdx.x;
      tdir[j] = a;
    }
  }
  if (threadIdx.x == 0) *head_cnt = (uint32_t)hc;
}

// the scoring kernel's 8-byte directory entry of every term (read once per index entry):
//   x = class << 30 | index   (sparse: first pair of the term; wide: batch-local wide id; head: hh)
//   y = pi_0 | pi_1 << 8 | pi_2 << 16 | min(queries, 255) << 24   (h <= 3, m <= 256)
// wide ids follow term order (wrank: exclusive scan of the wide flags), so a document's wide entries,
// walked in term order, come in wide-id order; terms past kNWMax wide ids stay sparse.  Head terms are
// re-marked by k_head_pick (their wide ids stay unused).
__global__ void k_ts_wflag(const uint32_t* __restrict__ qoff, int32_t n, int32_t wmin, uint32_t* __restrict__ flag) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    flag[j] = (int32_t)(qoff[j + 1] - qoff[j]) >= wmin ? 1u : 0u;
}

__global__ void k_ts_dir(const uint32_t* __restrict__ qoff, const uint16_t* __restrict__ pi, int32_t n, int32_t h,
                         int32_t wmin, const uint32_t* __restrict__ wrank, uint2* __restrict__ tdir,
                         uint32_t* __restrict__ wterm) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t qb = qoff[j], nq = qoff[j + 1] - qb;
    uint32_t y = 0;
    for (int o = 0; o < h; o++) y |= (uint32_t)pi[j * h + o] << (8 * o);
    y |= min(nq, 255u) << 24;
    uint32_t x = kClsAbsent << kClsShift;
    if (nq > 0) {
      x = (kClsSparse << kClsShift) | qb;
      if ((int32_t)nq >= wmin) {
        const uint32_t w = wrank[j];
        if (w < (uint32_t)kNWMax) {
          x = (kClsWide << kClsShift) | w;
          wterm[w] = (uint32_t)j;
        }
      }
    }
    tdir[j] = make_uint2(x, y);
  }
}

// one block: the wide-pair table in wide-id order (wpairs, wpoff[w] .. wpoff[w + 1]) and its groups —
// consecutive wide ids whose pairs fit the kernel's pair buffer together (gstart[g] .. gstart[g + 1])
__global__ void __launch_bounds__(1024) k_ts_wpairs(const uint32_t* __restrict__ qoff, const uint2* __restrict__ pairs,
                                                    const uint2* __restrict__ tdir, const uint32_t* __restrict__ wrank_n,
                                                    const uint32_t* __restrict__ wterm, uint32_t pb,
                                                    uint32_t* __restrict__ wpoff, uint32_t* __restrict__ gstart,
                                                    uint32_t* __restrict__ ngroups, uint2* __restrict__ wpairs) {
  __shared__ uint32_t cnt[kNWMax + 1], off[kNWMax + 1];
  const uint32_t nw = min(*wrank_n, (uint32_t)kNWMax);
  for (uint32_t w = threadIdx.x; w < (uint32_t)kNWMax; w += blockDim.x) {
    uint32_t c = 0;
    if (w < nw) {
      const uint32_t j = wterm[w];
      if ((tdir[j].x >> kClsShift) == kClsWide) c = qoff[j + 1] - qoff[j];  // (head terms: no pairs here)
    }
    cnt[w] = c;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t acc = 0, g = 0, in_g = 0;
    gstart[0] = 0;
    for (uint32_t w = 0; w < nw; w++) {
      if (in_g + cnt[w] > pb && in_g > 0) {
        gstart[++g] = w;
        in_g = 0;
      }
      off[w] = acc;
      acc += cnt[w];
      in_g += cnt[w];
    }
    off[nw] = acc;
    gstart[++g] = nw;
    *ngroups = nw ? g : 0;
  }
  __syncthreads();
  for (uint32_t w = threadIdx.x; w <= (uint32_t)kNWMax; w += blockDim.x) wpoff[w] = off[min(w, nw)];
  for (uint32_t w = 0; w < nw; w++) {
    if (!cnt[w]) continue;
    const uint32_t b = qoff[wterm[w]];
    for (uint32_t r = threadIdx.x; r < cnt[w]; r += blockDim.x) wpairs[off[w] + r] = pairs[b + r];
  }
}

// ---------------------------------------------------------------- the tile kernel
enum { kTsHist = 0, kTsEmit = 1 };

struct TsArgs {
  const int64_t* toff;
  const uint32_t* post;
  int64_t nunits;       // tiles visited: t = it * stride, it < nunits
  int64_t stride;
  const uint8_t* live;
  const int32_t* nnz;   // per-id entries stored in its tile (ecnt: tombstones of deleted ids included)
  const float* U;
  const float* L;       // null under Sinnamon+
  int32_t m;
  int32_t h;            // <= 3 (packed maps)
  const uint2* tdir;
  const uint32_t* qoff;
  const uint2* pairs;
  const uint32_t* wterm;   // [kNWMax] wide id -> term
  const float* Qh;         // [kTsHMax][kTQ]
  const uint32_t* head_cnt;
  int32_t nqc;
  const float* theta;      // EMIT: theta_q; HIST: a positive floor from a smaller nested sample (or null)
  unsigned long long* cand;
  uint32_t* cand_cnt;
  uint32_t cand_cap;
  uint32_t* hist;          // HIST: [nqc][kThetaBinsT]
  uint32_t* nsampled;
  uint32_t* sched;         // work-unit counter (zeroed before the launch)
  const uint32_t* allow;   // constrained search (Eq. 3): column mask, bit i of word i/32; null = all
  int64_t allow_words;
  int32_t hsm;             // head terms held in shared memory (QS == true): the Qs rows
  int32_t dw;              // wide entries per document listed for the wide pass
  const uint2* wpairs;     // wide pairs in wide-id order
  const uint32_t* wpoff;   // [kNWMax + 1]
  const uint32_t* gstart;  // groups of wide ids
  const uint32_t* ngroups;
  int32_t pbcap;           // pairs of the shared-memory pair buffer
  unsigned long long* prof;  // SINN_TS_PROF=1 (diagnostics): per CTA [8] phase clocks
};

__host__ __device__ inline int ts_sides(bool lower) { return lower ? 2 : 1; }

// shared-memory layout (bytes), in this order: S, sketch tile / pair buffer (one region: the pair
// buffer is used after the decode pass, the next tile's sketch streams in after the wide pass), Qs,
// E (head), tags, per-warp wide lists (wide id + decoded estimates of the warp's document), control
constexpr int kPbMin = 3072;       // pair-buffer capacity floor (pairs)
constexpr int kDocWidesMax = 128;  // wide entries per document kept for the wide pass (more: walked in B)
struct TsSmem {
  size_t S, col, qs, eh, tags, dlw, dle, wpo, ctl, total;
  int pbcap;
};

__host__ __device__ inline TsSmem ts_smem(int m, bool lower, int hsm, int dw) {
  TsSmem L;
  const int sides = ts_sides(lower);
  size_t o = 0;
  L.S = o;    o += sizeof(float) * kTD * kTQ;
  const size_t colb = sizeof(float) * (size_t)kTD * m * sides;
  const size_t pbb = colb > sizeof(uint2) * kPbMin ? colb : sizeof(uint2) * kPbMin;
  L.pbcap = (int)(pbb / sizeof(uint2));
  L.col = o;  o += pbb;
  L.qs = o;   o += sizeof(float) * (size_t)hsm * kTQ;
  L.eh = o;   o += sizeof(float) * (size_t)kTsHMax * sides * kTD;
  L.tags = o; o += (size_t)32 * kTags;
  L.dle = o;  o += sizeof(float) * (size_t)32 * dw * sides;
  L.dlw = o;  o += sizeof(uint16_t) * (size_t)32 * dw;
  o = (o + 15) & ~(size_t)15;
  L.wpo = o;  o += sizeof(uint32_t) * (kNWMax + 1);
  L.ctl = o;  o = ((o + 15) & ~(size_t)15) + 64;
  L.total = o;
  return L;
}

__device__ __forceinline__ void ts_cp16(void* sdst, const void* gsrc) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gsrc));
}
__device__ __forceinline__ void ts_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void ts_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

// the tile's sketch columns (32 consecutive ids: one contiguous block of U, one of L) -> col
template <bool LOWER>
__device__ __forceinline__ void ts_stage(const TsArgs& A, int64_t t, float* col) {
  const int64_t chunks = (int64_t)kTD * A.m / 4;  // 16-byte chunks per side (m % 4 == 0)
  const float4* gu = reinterpret_cast<const float4*>(A.U + t * kTD * A.m);
  for (int64_t c = threadIdx.x; c < chunks; c += blockDim.x) ts_cp16(col + 4 * c, gu + c);
  if (LOWER) {
    const float4* gl = reinterpret_cast<const float4*>(A.L + t * kTD * A.m);
    float* cl = col + (int64_t)kTD * A.m;
    for (int64_t c = threadIdx.x; c < chunks; c += blockDim.x) ts_cp16(cl + 4 * c, gl + c);
  }
  ts_commit();
}

__device__ __forceinline__ uint32_t ts_lanemask_lt() {
  uint32_t r;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
  return r;
}

// LOWER: the index keeps the lower sketch (two-sided, Sinnamon); QS: the head rows Q[hh][*] are held in
// shared memory (A.hsm rows), else read from global memory (L1/L2) in the dense phase, one term ahead.
template <int MODE, bool LOWER, bool QS>
__global__ void __launch_bounds__(1024, 1) k_ts_score(TsArgs A) {
  extern __shared__ float4 ts_smem4[];
  char* base = reinterpret_cast<char*>(ts_smem4);
  const TsSmem Lo = ts_smem(A.m, LOWER, QS ? A.hsm : 0, A.dw);
  float* S = reinterpret_cast<float*>(base + Lo.S);
  float* col = reinterpret_cast<float*>(base + Lo.col);
  uint2* pb = reinterpret_cast<uint2*>(base + Lo.col);  // the pair buffer (aliases the sketch tile)
  float* Qs = reinterpret_cast<float*>(base + Lo.qs);
  float* Eh = reinterpret_cast<float*>(base + Lo.eh);
  uint8_t* tags_all = reinterpret_cast<uint8_t*>(base + Lo.tags);
  uint32_t* ctl = reinterpret_cast<uint32_t*>(base + Lo.ctl);  // [0] next unit [3] tile live mask
  uint32_t* wpo = reinterpret_cast<uint32_t*>(base + Lo.wpo);  // wide-pair offsets of the pass (once per CTA)
  constexpr int SD = LOWER ? 2 : 1;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int m = A.m;
  const int nqc = A.nqc;
  const int hc = (int)*A.head_cnt;
  const int hn = QS ? min(hc, A.hsm) : min(hc, kTsHMax);
  const int ngroups = (int)*A.ngroups;
  uint8_t* tags = tags_all + w * kTags;
  const int dw = A.dw;
  uint16_t* dlist = reinterpret_cast<uint16_t*>(base + Lo.dlw) + w * dw;  // this warp's document: its wide ids,
  float* dle = reinterpret_cast<float*>(base + Lo.dle) + w * dw * SD;     // ascending, and their estimates
  // dense-phase mapping: thread = 2 queries x 16 documents (warp: 64 queries x one half of the tile)
  const int qp = ((w & 15) << 5) | lane;
  const int q0 = 2 * qp;
  const int dh = (w >> 4) * 16;
  if (QS)
    for (int t2 = tid; t2 < hn * kTQ; t2 += blockDim.x) Qs[t2] = A.Qh[t2];
  float th0, th1;  // EMIT: theta of the two queries (+inf past nqc); HIST: the floor (-inf: none)
  if (MODE == kTsEmit) {
    th0 = q0 < nqc ? A.theta[q0] : INFINITY;
    th1 = q0 + 1 < nqc ? A.theta[q0 + 1] : INFINITY;
  } else {
    const float f0 = (A.theta && q0 < nqc) ? A.theta[q0] : -INFINITY;
    const float f1 = (A.theta && q0 + 1 < nqc) ? A.theta[q0 + 1] : -INFINITY;
    th0 = f0 > 0.f ? f0 : -INFINITY;
    th1 = f1 > 0.f ? f1 : -INFINITY;
  }
  for (int i = tid; i < kTD * kTQ; i += blockDim.x) S[i] = 0.0f;
  for (int i = tid; i <= kNWMax; i += blockDim.x) wpo[i] = A.wpoff[i];
  if (tid == 0) ctl[0] = atomicAdd(A.sched, 1u);
  __syncthreads();
  int64_t u = ctl[0];
  if (u < A.nunits) ts_stage<LOWER>(A, u * A.stride, col);
  uint32_t nsampled = 0;
  auto sgn_est = [](float v, float a, float b) { return LOWER ? (v > 0.0f ? a : b) : a; };
  unsigned long long pc[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};  // (A.prof) phase clocks of thread 0 / warp busy sums
  long long c0 = clock64(), c1 = 0;
  while (u < A.nunits) {
    const int64_t t = u * A.stride;
    const int64_t tb = A.toff[t], te = A.toff[t + 1];
    // ---- head estimates zeroed; the live (and allowed) documents of the tile
    for (int i = tid; i < kTsHMax * SD * kTD; i += blockDim.x) Eh[i] = 0.0f;
    if (w == 0) {
      const bool lv = A.live[t * kTD + lane] != 0;
      uint32_t lm = __ballot_sync(kFullT, lv);
      if (A.allow) lm &= t < A.allow_words ? __ldg(A.allow + t) : 0u;
      if (lane == 0) ctl[3] = lm;
    }
    ts_wait_all();
    __syncthreads();
    if (A.prof) {
      c1 = clock64();
      pc[0] += c1 - c0;  // tile start -> decode start (the sketch wait)
      c0 = c1;
    }
    const uint32_t lmask = ctl[3];
    // ---- B: warp = document w: decode every batch-term entry from the staged column; head -> E,
    // wide -> this warp's list (wide id, estimates), the rest added into S now
    uint32_t ndl = 0;  // wide ids listed for the wide pass
    {
      const int d = w;
      const int64_t i_lane = t * kTD + lane;
      const uint32_t c_lane = (uint32_t)A.nnz[i_lane];  // entries stored (tombstones included)
      uint32_t inc = c_lane;
#pragma unroll
      for (int dd = 1; dd < 32; dd <<= 1) {
        const uint32_t y = __shfl_up_sync(kFullT, inc, dd);
        if (lane >= dd) inc += y;
      }
      const uint32_t cnt = __shfl_sync(kFullT, c_lane, d);
      const uint32_t e0 = __shfl_sync(kFullT, inc - c_lane, d);
      float* Srow = S + d * kTQ;
      const float* colU = col + d * m;
      const float* colL = col + kTD * m + d * m;
      const bool active = (lmask >> d) & 1u;
      // pipeline: the entries of chunk c + 2 and the directory words of chunk c + 1 are in flight
      // while chunk c is processed (no load is waited on where it is issued)
      auto ld_entry = [&](uint32_t c) -> uint32_t {
        return (active && c + lane < cnt) ? __ldg(A.post + tb + e0 + c + lane) : 0xffffffffu;
      };
      auto ld_dir = [&](uint32_t raw) -> uint2 {
        return raw != 0xffffffffu ? __ldg(A.tdir + (raw >> 5)) : make_uint2(0, 0);
      };
      uint32_t r_cur = ld_entry(0), r_nxt = ld_entry(32);
      uint2 d_cur = ld_dir(r_cur);
      for (uint32_t c0 = 0; active && c0 < cnt; c0 += 32) {
        const uint32_t j = r_cur == 0xffffffffu ? 0u : (r_cur >> 5);
        const uint32_t x = d_cur.x, y = d_cur.y;
        const uint32_t r_nn = ld_entry(c0 + 64);
        const uint2 d_nxt = ld_dir(r_nxt);
        r_cur = r_nxt;
        r_nxt = r_nn;
        d_cur = d_nxt;
        const uint32_t cls = x >> kClsShift;
        float eu = 0.f, el = 0.f;
        if (cls != kClsAbsent) {
          eu = colU[y & 0xffu];
          if (A.h > 1) eu = fminf(eu, colU[(y >> 8) & 0xffu]);
          if (A.h > 2) eu = fminf(eu, colU[(y >> 16) & 0xffu]);
          if (LOWER) {
            el = colL[y & 0xffu];
            if (A.h > 1) el = fmaxf(el, colL[(y >> 8) & 0xffu]);
            if (A.h > 2) el = fmaxf(el, colL[(y >> 16) & 0xffu]);
          }
        }
        uint32_t nr = 0, qb = 0;  // sparse pairs this lane walks here
        bool listed = false;
        if (cls == kClsHead) {
          const int hh = (int)(x & 0xffffu);
          Eh[(hh * SD) * kTD + d] = eu;
          if (LOWER) Eh[(hh * SD + 1) * kTD + d] = el;
        } else if (cls == kClsWide) {
          listed = true;
        } else if (cls == kClsSparse) {
          qb = x & 0x3fffffffu;
          nr = y >> 24;
          if (nr == 255u) nr = A.qoff[j + 1] - qb;
        }
        // the wide ids of this chunk, appended in entry (= term = wide-id) order
        const uint32_t lb = __ballot_sync(kFullT, listed);
        if (listed) {
          const uint32_t pos = ndl + __popc(lb & ts_lanemask_lt());
          if (pos < (uint32_t)dw) {
            dlist[pos] = (uint16_t)(x & 0xffffu);
            dle[pos * SD] = eu;
            if (LOWER) dle[pos * SD + 1] = el;
          } else {  // list full: this entry is walked here, warp-wide
            const uint32_t jj = A.wterm[x & 0xffffu];
            qb = A.qoff[jj];
            nr = A.qoff[jj + 1] - qb;
          }
        }
        ndl = min(ndl + __popc(lb), (uint32_t)dw);
        // every sparse pair load of the chunk is issued before any update (one L2 round trip per
        // chunk): the narrow lanes' <= 8 pairs into registers, and the first 32 pairs of up to four
        // warp-wide terms (> 8 queries; lane = pair)
        uint32_t wide = __ballot_sync(kFullT, nr > 8u);
        const uint32_t nrn = nr > 8u ? 0u : nr;
        uint2 np[8];
#pragma unroll
        for (int k = 0; k < 8; k++) np[k] = (uint32_t)k < nrn ? __ldg(A.pairs + qb + k) : make_uint2(0, 0);
        while (wide) {
          int srcs[4];
          uint2 wp[4];
          int nt = 0;
#pragma unroll
          for (int k = 0; k < 4; k++) {
            srcs[k] = -1;
            if (wide) {
              srcs[k] = __ffs(wide) - 1;
              wide &= wide - 1;
              nt++;
            }
            const int sk = srcs[k] < 0 ? 0 : srcs[k];
            const uint32_t b = __shfl_sync(kFullT, qb, sk), nn = srcs[k] < 0 ? 0u : __shfl_sync(kFullT, nr, sk);
            wp[k] = (uint32_t)lane < nn ? __ldg(A.pairs + b + lane) : make_uint2(0, 0);
          }
#pragma unroll
          for (int k = 0; k < 4; k++) {
            if (k >= nt) break;
            const int sk = srcs[k];
            const uint32_t b = __shfl_sync(kFullT, qb, sk), nn = __shfl_sync(kFullT, nr, sk);
            const float wu = __shfl_sync(kFullT, eu, sk), wl = __shfl_sync(kFullT, el, sk);
            if ((uint32_t)lane < nn) {  // a term's queries are distinct: no two lanes meet the same cell
              const float v = __uint_as_float(wp[k].y);
              Srow[wp[k].x] = fmaf(v, sgn_est(v, wu, wl), Srow[wp[k].x]);
            }
            for (uint32_t r = lane + 32; r < nn; r += 32) {  // terms past 32 pairs (spilled wide terms)
              const uint2 pr = __ldg(A.pairs + b + r);
              const float v = __uint_as_float(pr.y);
              Srow[pr.x] = fmaf(v, sgn_est(v, wu, wl), Srow[pr.x]);
            }
            __syncwarp();  // two terms may share a query
          }
        }
        // narrow terms: lane = entry, serial over its <= 8 pairs; lanes meeting the same query
        // (a query sharing two terms with the document) are serialised through the tag bytes
        const uint32_t maxr = __reduce_max_sync(kFullT, nrn);
#pragma unroll
        for (int r = 0; r < 8; r++) {
          if ((uint32_t)r >= maxr) break;
          bool pend = (uint32_t)r < nrn;
          const uint32_t q = np[r].x & (kTQ - 1);
          const float v = __uint_as_float(np[r].y);
          const float add = v * sgn_est(v, eu, el);
          while (__any_sync(kFullT, pend)) {
            if (pend) tags[q & (kTags - 1)] = (uint8_t)lane;
            __syncwarp();
            const bool win = pend && tags[q & (kTags - 1)] == (uint8_t)lane;
            if (win) Srow[q] += add;
            pend = pend && !win;
            __syncwarp();
          }
        }
      }
    }
    if (A.prof && lane == 0) pc[5] += clock64() - c0;  // this warp's busy time in B
    if (tid == 0) ctl[0] = atomicAdd(A.sched, 1u);  // the next unit
    __syncthreads();
    if (A.prof) {
      c1 = clock64();
      pc[1] += c1 - c0;  // decode + sparse pass (wall)
      c0 = c1;
    }
    const int64_t un = ctl[0];
    // ---- C: wide terms.  Their pairs are staged group by group in the pair buffer (loaded once per
    // tile for all its documents); warp w adds the terms of its own document into its own row only
    // (race-free: a row has one writer), walking its wide-id list in step with the groups.
    {
      const int d = w;
      const bool active = (lmask >> d) & 1u;
      float* Srow = S + d * kTQ;
      uint32_t cur = 0;  // position in this warp's list
      for (int g = 0; g < ngroups; g++) {
        const uint32_t w0 = A.gstart[g], w1 = A.gstart[g + 1];
        const uint32_t p0 = wpo[w0], p1 = wpo[w1];
        // the group's pairs -> the pair buffer: asynchronous 8-byte copies, all in flight at once
        for (uint32_t i = tid; i < p1 - p0; i += blockDim.x) {
          const uint32_t sa = (uint32_t)__cvta_generic_to_shared(pb + i);
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(A.wpairs + p0 + i));
        }
        ts_commit();
        ts_wait_all();
        __syncthreads();
        long long cg = A.prof ? clock64() : 0;
        while (active && cur < ndl) {
          const uint32_t wid = dlist[cur];
          if (wid >= w1) break;
          float eu, el = 0.f;
          if (LOWER) {
            const float2 e2 = *reinterpret_cast<const float2*>(dle + 2 * cur);
            eu = e2.x;
            el = e2.y;
          } else {
            eu = dle[cur];
          }
          cur++;
          const uint32_t a0 = wpo[wid] - p0, nn = wpo[wid + 1] - wpo[wid];
          // four independent read-modify-writes per lane in flight (distinct queries within a term)
          for (uint32_t r = lane; r < nn; r += 128) {
            uint2 pr[4];
#pragma unroll
            for (int k = 0; k < 4; k++) pr[k] = r + 32 * k < nn ? pb[a0 + r + 32 * k] : make_uint2(0, 0);
            float sv[4];
#pragma unroll
            for (int k = 0; k < 4; k++) sv[k] = Srow[pr[k].x];
#pragma unroll
            for (int k = 0; k < 4; k++) {
              const float v = __uint_as_float(pr[k].y);
              if (r + 32 * k < nn) Srow[pr[k].x] = fmaf(v, sgn_est(v, eu, el), sv[k]);
            }
          }
        }
        if (A.prof && lane == 0) {
          pc[8] += clock64() - cg;  // this warp's busy time in the group
          if (w == 0) pc[9] += 1;
        }
        __syncthreads();
      }
    }
    if (A.prof) {
      c1 = clock64();
      pc[2] += c1 - c0;  // wide pass (wall)
      c0 = c1;
    }
    if (un < A.nunits) ts_stage<LOWER>(A, un * A.stride, col);  // the next tile's sketch streams in from here
    // ---- C': this warp's block of the dense head product (registers): 16 documents x 2 queries
    float acc[16][2];
#pragma unroll
    for (int d = 0; d < 16; d++) acc[d][0] = acc[d][1] = 0.f;
    float2 qn2 = make_float2(0.f, 0.f);
    if (!QS && hn > 0) qn2 = __ldg(reinterpret_cast<const float2*>(A.Qh + q0));
    for (int hh = 0; hh < hn; hh++) {
      float qa, qb2;
      if (QS) {
        const float2 v = *reinterpret_cast<const float2*>(Qs + hh * kTQ + q0);
        qa = v.x;
        qb2 = v.y;
      } else {  // one term ahead from L1/L2
        qa = qn2.x;
        qb2 = qn2.y;
        if (hh + 1 < hn) qn2 = __ldg(reinterpret_cast<const float2*>(A.Qh + (hh + 1) * kTQ + q0));
      }
      const float4* ep = reinterpret_cast<const float4*>(Eh + (hh * SD) * kTD + dh);
      if (LOWER) {
        const float4* en = reinterpret_cast<const float4*>(Eh + (hh * SD + 1) * kTD + dh);
        const float pa = fmaxf(qa, 0.f), na = fminf(qa, 0.f), pb2 = fmaxf(qb2, 0.f), nb = fminf(qb2, 0.f);
#pragma unroll
        for (int k = 0; k < 4; k++) {
          const float4 u4 = ep[k], l4 = en[k];
          const float uu[4] = {u4.x, u4.y, u4.z, u4.w}, ll[4] = {l4.x, l4.y, l4.z, l4.w};
#pragma unroll
          for (int c = 0; c < 4; c++) {
            acc[4 * k + c][0] = fmaf(na, ll[c], fmaf(pa, uu[c], acc[4 * k + c][0]));
            acc[4 * k + c][1] = fmaf(nb, ll[c], fmaf(pb2, uu[c], acc[4 * k + c][1]));
          }
        }
      } else {
#pragma unroll
        for (int k = 0; k < 4; k++) {
          const float4 u4 = ep[k];
          const float uu[4] = {u4.x, u4.y, u4.z, u4.w};
#pragma unroll
          for (int c = 0; c < 4; c++) {
            acc[4 * k + c][0] = fmaf(qa, uu[c], acc[4 * k + c][0]);
            acc[4 * k + c][1] = fmaf(qb2, uu[c], acc[4 * k + c][1]);
          }
        }
      }
    }
    if (A.prof && lane == 0) pc[6] += clock64() - c0;  // this warp's busy time in the dense block
    __syncthreads();
    if (A.prof) {
      c1 = clock64();
      pc[3] += c1 - c0;  // dense head (wall)
      c0 = c1;
    }
    // ---- D: S + head product vs theta; S reset; wide bytes reset
    {
      const uint32_t lm = lmask >> dh;
      const int64_t id0 = t * kTD + dh;
#pragma unroll
      for (int d = 0; d < 16; d++) {
        float2* cell = reinterpret_cast<float2*>(S + (dh + d) * kTQ + q0);
        const float2 sv = *cell;
        *cell = make_float2(0.f, 0.f);
        if (!((lm >> d) & 1u)) continue;
        float x0 = sv.x + acc[d][0], x1 = sv.y + acc[d][1];
        if (x0 == 0.0f) x0 = 0.0f;  // -0.0 -> +0.0 (R19)
        if (x1 == 0.0f) x1 = 0.0f;
        const uint32_t id = (uint32_t)(id0 + d);
        if (MODE == kTsEmit) {
          if (x0 >= th0) {
            const uint32_t pos = atomicAdd(&A.cand_cnt[q0], 1u);
            if (pos < A.cand_cap)
              A.cand[(int64_t)q0 * A.cand_cap + pos] = ((unsigned long long)f2key(x0) << 32) | (unsigned long long)(~id);
          }
          if (x1 >= th1) {
            const uint32_t pos = atomicAdd(&A.cand_cnt[q0 + 1], 1u);
            if (pos < A.cand_cap)
              A.cand[(int64_t)(q0 + 1) * A.cand_cap + pos] =
                  ((unsigned long long)f2key(x1) << 32) | (unsigned long long)(~id);
          }
        } else {
          if (q0 < nqc && x0 != 0.0f && x0 >= th0)
            atomicAdd(&A.hist[(int64_t)q0 * kThetaBinsT + (f2key(x0) >> kThetaShiftT)], 1u);
          if (q0 + 1 < nqc && x1 != 0.0f && x1 >= th1)
            atomicAdd(&A.hist[(int64_t)(q0 + 1) * kThetaBinsT + (f2key(x1) >> kThetaShiftT)], 1u);
        }
      }
      if (MODE == kTsHist && tid == 0) nsampled += __popc(lmask);
    }
    __syncthreads();
    if (A.prof) {
      c1 = clock64();
      pc[4] += c1 - c0;  // epilogue (wall)
      c0 = c1;
      pc[7] += 1;
    }
    u = un;
  }
  if (A.prof && lane == 0) {
    if (tid == 0)
      for (int k = 0; k < 5; k++) atomicAdd(&A.prof[k], pc[k]);
    atomicAdd(&A.prof[5], pc[5]);
    atomicAdd(&A.prof[6], pc[6]);
    atomicAdd(&A.prof[8], pc[8]);
    if (tid == 0) atomicAdd(&A.prof[7], pc[7]);
    if (tid == 0) atomicAdd(&A.prof[9], pc[9]);
  }
  ts_wait_all();
  if (MODE == kTsHist && tid == 0 && nsampled) atomicAdd(A.nsampled, nsampled);
}

template <int MODE, bool LOWER, bool QS>
void ts_go(const TsArgs& A, size_t smem, cudaStream_t s) {
  auto kern = k_ts_score<MODE, LOWER, QS>;
  smem_optin((const void*)kern);
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(sm_count(), A.nunits));
  kern<<<grid, 1024, smem, s>>>(A);
}

}  // namespace

// ---------------------------------------------------------------- host side
// dynamic shared memory the layout may use: the sm_100 per-block opt-in maximum (227 KB) less 1 KB
// for the kernel's static shared memory (the scan's warp totals)
constexpr size_t kTsSmemBudget = 227 * 1024 - 1024;

bool ts_supported(int m, int h, bool lower, bool bf16) {
  if (bf16 || h > 3 || m > 256 || (m & 3) != 0) return false;
  return ts_smem(m, lower, 0, 32).total <= kTsSmemBudget;
}

// head rows held in shared memory (next to an estimate list of 2,048 slots); below 8 rows the rows are
// read from global memory instead (QS == false) and up to kTsHMax head terms are taken
int ts_head_smem_rows(int m, bool lower) {
  const size_t fixed = ts_smem(m, lower, 0, 96).total;  // next to lists of 96 wide entries per document
  const size_t room = kTsSmemBudget > fixed ? kTsSmemBudget - fixed : 0;
  const int r = (int)std::min<size_t>(kTsHMax, room / (sizeof(float) * kTQ));
  return r >= 8 ? r : 0;
}

int ts_head_max(int m, bool lower) {
  const int r = ts_head_smem_rows(m, lower);
  return r ? r : kTsHMax;
}

// wide entries listed per document: what shared memory leaves next to the head rows (at most 128)
int ts_doc_wides(int m, bool lower, int hsm) {
  const size_t fixed = ts_smem(m, lower, hsm, 0).total;
  const size_t room = kTsSmemBudget > fixed ? kTsSmemBudget - fixed : 0;
  const size_t per = (size_t)32 * (sizeof(uint16_t) + sizeof(float) * ts_sides(lower));
  return (int)std::min<size_t>(kDocWidesMax, room / per);
}

int ts_nwmax() { return kNWMax; }
int ts_hcand_cap() { return kHCand; }

void launch_head_select(const uint32_t* qoff, const int32_t* df, int32_t n, int64_t live, int64_t nq, float tau,
                        const uint2* pairs, uint4* dir, uint2* tdir, float* Qh, uint32_t* head_cnt,
                        unsigned long long* hcand, uint32_t* nhcand, int hmax, int qrow, cudaStream_t s) {
  cudaMemsetAsync(nhcand, 0, sizeof(uint32_t), s);
  const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)sm_count() * 8));
  k_head_cand<<<blocks, 256, 0, s>>>(qoff, df, n, 1.0f / (float)std::max<int64_t>(live, 1),
                                     1.0f / (float)std::max<int64_t>(nq, 1), tau, hcand, nhcand);
  k_head_pick<<<1, 1024, 0, s>>>(hcand, nhcand, qoff, pairs, dir, tdir, Qh, head_cnt, std::min(hmax, kTsHMax), qrow);
}

void launch_ts_dir(const uint32_t* qoff, const uint16_t* pi, int32_t n, int32_t h, int32_t wmin, uint2* tdir,
                   uint32_t* wflag, uint32_t* wrank, uint32_t* scan_tmp, uint32_t* wterm, cudaStream_t s) {
  const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)sm_count() * 8));
  k_ts_wflag<<<blocks, 256, 0, s>>>(qoff, n, wmin, wflag);
  cudaMemsetAsync(wflag + n, 0, sizeof(uint32_t), s);
  exclusive_scan_u32(wflag, wrank, n + 1, scan_tmp, s);  // wrank[n] = wide terms of the pass
  k_ts_dir<<<blocks, 256, 0, s>>>(qoff, pi, n, h, wmin, wrank, tdir, wterm);
}

int ts_pair_buffer(int m, bool lower) { return ts_smem(m, lower, 0, 0).pbcap; }

void launch_ts_wpairs(const uint32_t* qoff, const uint2* pairs, const uint2* tdir, const uint32_t* wrank_n,
                      const uint32_t* wterm, int pbcap, uint32_t* wpoff, uint32_t* gstart, uint32_t* ngroups,
                      uint2* wpairs, cudaStream_t s) {
  k_ts_wpairs<<<1, 1024, 0, s>>>(qoff, pairs, tdir, wrank_n, wterm, (uint32_t)pbcap, wpoff, gstart, ngroups, wpairs);
}

void launch_ts_score(bool emit, const int64_t* toff, const uint32_t* post, int64_t ntiles_total, int64_t stride,
                     const uint8_t* live, const int32_t* nnz, const float* U, const float* L, int32_t m, int32_t h,
                     const uint2* tdir, const uint32_t* qoff, const uint2* pairs, const uint32_t* wterm,
                     const float* Qh, const uint32_t* head_cnt, int32_t hsm, int32_t nqc, const float* theta,
                     unsigned long long* cand, uint32_t* cand_cnt, uint32_t cand_cap, uint32_t* hist,
                     uint32_t* nsampled, uint32_t* sched, const uint32_t* allow, int64_t allow_words,
                     const uint2* wpairs, const uint32_t* wpoff, const uint32_t* gstart, const uint32_t* ngroups,
                     cudaStream_t s) {
  const bool lower = L != nullptr;
  const int hrows = ts_head_smem_rows(m, lower);  // 0: head rows from global memory
  TsArgs A{toff, post, (ntiles_total + stride - 1) / stride, stride, live, nnz, U, L, m, h, tdir, qoff, pairs, wterm, Qh,
           head_cnt, nqc, theta, cand, cand_cnt, cand_cap, hist, nsampled, sched, allow, allow_words,
           hrows ? std::min(hsm, hrows) : 0, 0, wpairs, wpoff, gstart, ngroups, 0, nullptr};
  A.dw = ts_doc_wides(m, lower, A.hsm);
  if (const char* e = getenv("SINN_TS_DOCWIDES")) A.dw = std::max(0, std::min(A.dw, atoi(e)));  // (overflow tests)
  const TsSmem Lo = ts_smem(m, lower, A.hsm, A.dw);
  A.pbcap = Lo.pbcap;
  cudaMemsetAsync(sched, 0, sizeof(uint32_t), s);
  static unsigned long long* prof = nullptr;
  const bool profon = getenv("SINN_TS_PROF") && getenv("SINN_TS_PROF")[0] == '1';
  if (profon) {
    if (!prof) cudaMalloc(&prof, 10 * sizeof(unsigned long long));
    cudaMemsetAsync(prof, 0, 10 * sizeof(unsigned long long), s);
    A.prof = prof;
  }
  const bool qs = A.hsm > 0;
#define SINN_TS_GO(MO)                                                              \
  {                                                                                 \
    if (lower) {                                                                    \
      if (qs) ts_go<MO, true, true>(A, Lo.total, s); else ts_go<MO, true, false>(A, Lo.total, s);   \
    } else {                                                                        \
      if (qs) ts_go<MO, false, true>(A, Lo.total, s); else ts_go<MO, false, false>(A, Lo.total, s); \
    }                                                                               \
  }
  if (emit) SINN_TS_GO(kTsEmit) else SINN_TS_GO(kTsHist)
#undef SINN_TS_GO
  if (profon) {  // diagnostics: mean clocks per tile of each phase (wall) and the warps' mean busy time
    unsigned long long h[10];
    cudaMemcpyAsync(h, prof, sizeof(h), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    const double nt = h[7] ? (double)h[7] : 1.0;
    fprintf(stderr, "[ts %s] tiles %llu  per tile: wait %.0f  decode+sparse %.0f (warp busy %.0f)  wide %.0f  dense %.0f "
            "(warp busy %.0f)  epilogue %.0f clocks; wide groups/tile %.1f, warp busy in groups %.0f\n",
            emit ? "emit" : "hist", h[7], h[0] / nt, h[1] / nt, h[5] / nt / 32, h[2] / nt, h[3] / nt, h[6] / nt / 32,
            h[4] / nt, h[9] / nt, h[8] / nt / 32);
  }
}

}  // namespace sinn
