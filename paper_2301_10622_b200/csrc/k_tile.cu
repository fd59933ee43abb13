// k_tile.cu — the scoring hot path (Alg. 6 + FindLargest k', T = infinity) for a batch of up to
// 1024 queries, over the tile-major inverted index (32-id tiles; inside a tile the incidence
// entries (j << 5) | d are grouped by document d).
//
//   k_qtab_count/fill  query prep (S0): the batch regrouped term-major — for every term j the
//                      (query, q_j) pairs with q_j != 0 (q_j > 0 only under Sinnamon+), and a
//                      16-byte directory entry per term: pair range, which signs occur, pi_o(j)
//   k_doc_score        persistent; each WARP owns one document at a time and its score row
//                      S[1024 queries] in shared memory, so no two threads ever update the same
//                      (document, query) cell concurrently: updates are plain LDS/FADD/STS (fp32
//                      atomicAdd on shared memory is an LDS + ATOMS.CAST CAS loop on sm_100a).
//                      Per document: its sketch column is staged in the warp's shared slot, its
//                      entries are walked 32 at a time (lane = entry), each present term is
//                      decoded once per needed sign, and q_j * e is added into S[q] for every
//                      query q of the term (lanes hitting the same q in one step are serialised
//                      by a per-warp tag array).  Terms with many queries are walked by the whole
//                      warp (lane = query; distinct queries, conflict-free).  Then the touched
//                      cells (or the whole row) are compared with theta_q and reset.
//                      HIST mode (sample pass, every stride-th tile): histograms the scores;
//                      EMIT mode keeps only scores >= theta_q, a provable lower bound of the
//                      k'-th largest score.
//   k_theta            theta_q = lower edge of the histogram bin holding the k'-th largest score
//                      of the sample (the k'-th largest of a subset never exceeds that of the set)
//   k_cand_select      exact top-k' of each query's candidates (radix select on the score key,
//                      then a bitonic sort of the survivors; ties by ascending id)
#include <math.h>

#include <stdlib.h>

#include <algorithm>

#include "k_doc.cuh"

namespace sinn {

namespace {

// ---------------------------------------------------------------- S0: batch term table
// anytime budget (Alg. 6 with T; R20): entry p of a query row is kept iff fewer
// than max_terms non-zero entries precede it in the (|q_j| desc, j asc) order (max_terms 0 = all)
__device__ __forceinline__ bool within_budget(const int32_t* __restrict__ qi, const float* __restrict__ qv,
                                              int64_t b, int64_t e, int64_t p, int32_t max_terms) {
  if (max_terms <= 0) return true;
  const float a = fabsf(qv[p]);
  const int32_t j = qi[p];
  int32_t rank = 0;
  for (int64_t r = b; r < e && rank < max_terms; r++) {
    const float ar = fabsf(qv[r]);
    rank += (ar != 0.0f) && (ar > a || (ar == a && qi[r] < j));
  }
  return rank < max_terms;
}

__global__ void k_qtab_count(const int64_t* __restrict__ q_indptr, const int32_t* __restrict__ q_indices,
                             const float* __restrict__ q_values, const int32_t* __restrict__ qlist, int64_t q0,
                             int64_t G, int32_t n, int upper_only, uint32_t* __restrict__ cnt,
                             uint32_t* __restrict__ sgn, uint32_t* __restrict__ bm, int32_t max_terms,
                             DevInfo* info) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  uint32_t err = 0;
  for (int64_t g = warp; g < G; g += nwarps) {
    const int64_t qi = qlist ? qlist[g] : q0 + g;
    const int64_t b = q_indptr[qi], e = q_indptr[qi + 1];
    if (e < b) {
      err |= kErrIndptr;
      continue;
    }
    for (int64_t p = b + lane; p < e; p += 32) {
      const int32_t j = q_indices[p];
      const float v = q_values[p];
      const bool bad = j < 0 || j >= n || !isfinite(v) || (p > b && q_indices[p - 1] >= j);
      if (bad) {
        err |= kErrRow;
        continue;
      }
      if (v == 0.0f || (upper_only && v < 0.0f)) continue;  // nz(q); Sinnamon+ (R6)
      if (!within_budget(q_indices, q_values, b, e, p, max_terms)) continue;
      atomicAdd(&cnt[j], 1u);
      if (sgn) atomicOr(&sgn[j], v > 0.0f ? 1u : 2u);
      if (bm) atomicOr(&bm[(int64_t)j * 32 + (g >> 5)], 1u << (g & 31));
    }
  }
  err = __reduce_or_sync(kFull, err);
  if (lane == 0 && err) atomicOr(&info->err, err);
}

__global__ void k_qtab_fill(const int64_t* __restrict__ q_indptr, const int32_t* __restrict__ q_indices,
                            const float* __restrict__ q_values, const int32_t* __restrict__ qlist, int64_t q0,
                            int64_t G, int32_t n, int upper_only, const uint32_t* __restrict__ qoff,
                            uint32_t* __restrict__ cursor, uint2* __restrict__ pairs, uint32_t pair_cap,
                            const uint32_t* __restrict__ bm, int32_t max_terms, DevInfo* info) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  if (warp == 0 && lane == 0 && qoff[n] > pair_cap) atomicOr(&info->pad, 1u);  // pair table overflow
  for (int64_t g = warp; g < G; g += nwarps) {
    const int64_t qi = qlist ? qlist[g] : q0 + g;
    const int64_t b = q_indptr[qi], e = q_indptr[qi + 1];
    for (int64_t p = b + lane; p < e; p += 32) {
      const int32_t j = q_indices[p];
      const float v = q_values[p];
      const bool bad = j < 0 || j >= n || !isfinite(v) || (p > b && q_indices[p - 1] >= j);
      if (bad || v == 0.0f || (upper_only && v < 0.0f)) continue;
      if (!within_budget(q_indices, q_values, b, e, p, max_terms)) continue;
      // with the query bitmap of term j (batches of <= 1024 queries) the pair's place is a pure
      // function of the term's query set (deterministic): narrow terms in query order; wide terms
      // (walked by the whole warp, lane = pair) bank-major, so that each 32-pair block holds
      // distinct score-row banks (q & 31) wherever the term has enough banks: the pair of query g
      // (bank bk, the r-th of the term's queries in that bank) goes after every pair of rank < r
      // and after the rank-r pairs of lower banks
      uint32_t rank;
      if (bm) {
        const uint32_t* b = bm + (int64_t)j * 32;
        const int wg = (int)(g >> 5), bk = (int)(g & 31);
        uint32_t words[32], nn = 0, r = 0;
#pragma unroll
        for (int w2 = 0; w2 < 32; w2++) {
          words[w2] = b[w2];
          nn += __popc(words[w2]);
          if (w2 < wg) r += (words[w2] >> bk) & 1u;
        }
        if (nn <= (uint32_t)kNarrowMax) {
          rank = __popc(words[wg] & ((1u << bk) - 1u));
#pragma unroll
          for (int w2 = 0; w2 < 32; w2++)
            if (w2 < wg) rank += __popc(words[w2]);
        } else {
          rank = 0;
#pragma unroll 4
          for (int b2 = 0; b2 < 32; b2++) {
            uint32_t cnt = 0;
#pragma unroll
            for (int w2 = 0; w2 < 32; w2++) cnt += (words[w2] >> b2) & 1u;
            rank += min(cnt, r) + ((b2 < bk && cnt > r) ? 1u : 0u);
          }
        }
      } else {
        rank = atomicAdd(&cursor[j], 1u);
      }
      const uint32_t pos = qoff[j] + rank;
      if (pos < pair_cap) pairs[pos] = make_uint2((uint32_t)g, __float_as_uint(v));
    }
  }
}

// directory entry of term j (32 bytes, one sector): dir[2j] = {first pair, end pair | has-positive
// << 30 | has-negative << 31, pi_0 | pi_1 << 16, pi_2 | pi_3 << 16} (h > 4 reads the table);
// dir[2j+1] = the term's first three (query, q_j) pairs inline: {q0 | q1 << 10 | q2 << 20, v0, v1, v2}
// (queries < 1024: bit 31 stays clear; a head term's entry is re-marked by k_head_pick), so most
// terms of a batch (few queries each) need no second lookup
__global__ void k_dir_fill(const uint32_t* __restrict__ qoff, const uint32_t* __restrict__ sgn,
                           const uint16_t* __restrict__ pi, const uint2* __restrict__ pairs, int32_t n, int32_t h,
                           uint32_t pair_cap, uint4* __restrict__ dir) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    uint32_t qb = qoff[j], qe = qoff[j + 1];
    if (qe > pair_cap) qe = qb = 0;  // overflowed table: the caller retries with a larger one
    uint32_t c[4] = {0, 0, 0, 0};
    for (int o = 0; o < h && o < 4; o++) c[o] = pi[j * h + o];
    const uint32_t s = sgn[j];
    dir[2 * j] = make_uint4(qb, qe | ((s & 1u) << 30) | ((s >> 1) << 31), c[0] | (c[1] << 16), c[2] | (c[3] << 16));
    uint2 p0 = make_uint2(0, 0), p1 = make_uint2(0, 0), p2 = make_uint2(0, 0);
    if (qe > qb) p0 = pairs[qb];
    if (qe > qb + 1) p1 = pairs[qb + 1];
    if (qe > qb + 2) p2 = pairs[qb + 2];
    dir[2 * j + 1] = make_uint4(p0.x | (p1.x << 10) | (p2.x << 20), p0.y, p1.y, p2.y);
  }
}


// ---------------------------------------------------------------- theta
// one CTA per query, thread t owning bins [32t, 32t + 32) (eight 16-byte loads): the bin of the
// k'-th largest sample score -> its lower edge (a provable bound).  The histogram holds the
// non-zero sample scores; zero scores = sampled - non-zero, counted in the bin of +0.0.
constexpr int kThetaThreads = kThetaBins / 32;
__global__ void __launch_bounds__(kThetaThreads) k_theta(const uint32_t* __restrict__ hist,
                                                          const uint32_t* __restrict__ nsampled, int nqc,
                                                          int kprime, float* __restrict__ theta,
                                                          uint32_t* __restrict__ list_ok,
                                                          const uint32_t* __restrict__ nsamp_q) {
  __shared__ uint32_t wsum[kThetaThreads / 32];
  const int q = blockIdx.x, t = threadIdx.x, lane = t & 31, w = t >> 5;
  if (q >= nqc) return;
  const uint4* h4 = reinterpret_cast<const uint4*>(hist + (int64_t)q * kThetaBins) + t * 8;
  uint32_t bin[32];
#pragma unroll
  for (int i = 0; i < 8; i++) {
    const uint4 v = h4[i];
    bin[4 * i] = v.x;
    bin[4 * i + 1] = v.y;
    bin[4 * i + 2] = v.z;
    bin[4 * i + 3] = v.w;
  }
  uint32_t mine = 0;
#pragma unroll
  for (int i = 0; i < 32; i++) mine += bin[i];
  // total non-zero sample scores of the query
  const uint32_t wtot = __reduce_add_sync(kFull, mine);
  if (lane == 0) wsum[w] = wtot;
  __syncthreads();
  uint32_t nonzero = 0, above_w = 0;
#pragma unroll
  for (int k = 0; k < kThetaThreads / 32; k++) {
    nonzero += wsum[k];
    if (k > w) above_w += wsum[k];
  }
  const uint32_t total = nsamp_q ? nsamp_q[q] : *nsampled;  // (F4: the query's own sample size)
  if (total < (uint32_t)kprime) {  // the sample cannot bound k': every live document is a candidate
    if (t == 0) {
      theta[q] = -INFINITY;
      *list_ok = 0u;
    }
    return;
  }
  const uint32_t zq = total - nonzero;
  const int zbin = (int)(f2key(0.0f) >> kThetaShift);
  if ((zbin >> 5) == t) {
#pragma unroll
    for (int i = 0; i < 32; i++)
      if (i == (zbin & 31)) bin[i] += zq;
    mine += zq;
  }
  // samples in bins above this thread's: the warp's higher lanes (suffix scan) + higher warps
  uint32_t inc = mine;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t v = __shfl_down_sync(kFull, inc, d);
    if (lane + d < 32) inc += v;
  }
  // (the zero count joined after the warp totals: warps below the zero bin's warp add it here)
  const uint32_t above = above_w + (inc - mine) + ((zbin >> 10) > w ? zq : 0u);
  if (above < (uint32_t)kprime && above + mine >= (uint32_t)kprime) {
    uint32_t acc = above;
    int b = 32 * t;
    bool found = false;
#pragma unroll
    for (int i = 31; i >= 0; i--) {
      if (!found) {
        acc += bin[i];
        if (acc >= (uint32_t)kprime) {
          found = true;
          b = 32 * t + i;
        }
      }
    }
    const float th = key2f((uint32_t)b << kThetaShift);
    theta[q] = th;
    if (!(th > 0.0f)) *list_ok = 0u;
  }
}

// ---------------------------------------------------------------- exact top-k' of the candidates
__device__ void bitonic_desc_u64(unsigned long long* s, int N) {
  for (int k = 2; k <= N; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      __syncthreads();
      for (int i = threadIdx.x; i < N; i += blockDim.x) {
        const int l = i ^ j;
        if (l > i) {
          const unsigned long long a = s[i], b = s[l];
          const bool up = (i & k) == 0;
          if (up ? (a < b) : (a > b)) {
            s[i] = b;
            s[l] = a;
          }
        }
      }
    }
  }
  __syncthreads();
}

// block-wide sum of one value per thread (NT threads); every thread gets the total
template <int NT>
__device__ __forceinline__ uint32_t block_sum(uint32_t n, uint32_t* wsum) {
  n = __reduce_add_sync(kFull, n);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = n;
  __syncthreads();
  uint32_t tot = (threadIdx.x & 31) < (NT >> 5) ? wsum[threadIdx.x & 31] : 0u;
  tot = __reduce_add_sync(kFull, tot);
  __syncthreads();
  return tot;
}

// k_cand_select's register path: K = the target-th largest score key among c[0..cnt) (each of the
// NT threads holds PER keys), found bit by bit with block-wide counts.  Every candidate with key > K
// is taken; the ties of K are taken whole when they fit the sort buffer, else only the ones with the
// smallest ids (a second bitwise select on the low word ~id among key == K: the composite order
// (score desc, id asc) of sinn.h and DESIGN.md R10, never the atomic arrival order).  Returns the
// bitonic size (power of two >= the count copied to sb).
template <int PER, int NT>
__device__ int reg_select(const unsigned long long* __restrict__ c, uint32_t cnt, uint32_t target, int sort_cap,
                          unsigned long long* sb, uint32_t* s_count, uint32_t* s_ties) {
  __shared__ uint32_t wsum[32];
  uint32_t keys[PER];
#pragma unroll
  for (int i = 0; i < PER; i++) {
    const uint32_t t = threadIdx.x + (uint32_t)NT * i;
    keys[i] = t < cnt ? (uint32_t)(c[t] >> 32) : 0u;  // key 0 (below every finite score) = empty
  }
  uint32_t K = 0;
  for (int bit = 31; bit >= 0; bit--) {
    const uint32_t trial = K | (1u << bit);
    uint32_t n = 0;
#pragma unroll
    for (int i = 0; i < PER; i++) n += keys[i] >= trial ? 1u : 0u;
    if (block_sum<NT>(n, wsum) >= target) K = trial;
  }
  uint32_t na = 0, nt = 0;
#pragma unroll
  for (int i = 0; i < PER; i++) {
    na += keys[i] > K ? 1u : 0u;
    nt += keys[i] == K ? 1u : 0u;
  }
  const uint32_t above = block_sum<NT>(na, wsum), ties = block_sum<NT>(nt, wsum);
  // low-word (~id) threshold among the ties: 0 takes every tie
  uint32_t Lw = 0;
  if (above + ties > (uint32_t)sort_cap) {
    const uint32_t need = target - above;  // >= 1
    for (int bit = 31; bit >= 0; bit--) {
      const uint32_t trial = Lw | (1u << bit);
      uint32_t n = 0;
#pragma unroll
      for (int i = 0; i < PER; i++) {
        const uint32_t t = threadIdx.x + (uint32_t)NT * i;
        if (keys[i] == K && t < cnt && (uint32_t)c[t] >= trial) n++;
      }
      if (block_sum<NT>(n, wsum) >= need) Lw = trial;
    }
  }
  if (threadIdx.x == 0) {
    *s_count = 0;
    *s_ties = 0;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < PER; i++) {
    const uint32_t t = threadIdx.x + (uint32_t)NT * i;
    if (t < cnt && keys[i] >= K) {
      const unsigned long long v = c[t];
      if (keys[i] > K || (uint32_t)v >= Lw) {
        const uint32_t pos = atomicAdd(s_count, 1u);
        if (pos < (uint32_t)sort_cap) sb[pos] = v;
      }
    }
  }
  __syncthreads();
  const int got = (int)min(*s_count, (uint32_t)sort_cap);
  int N = 1;
  while (N < got) N <<= 1;
  for (int t = got + threadIdx.x; t < N; t += blockDim.x) sb[t] = 0ull;
  return N;
}

// One CTA per query.  A candidate is (score key << 32) | ~id, so the u64 order is (score desc,
// id asc).  Radix select (12/12/8 bits of the score key) finds the key K of the target-th largest;
// every candidate with key >= K is collected (all ties of K while they fit) and bitonic-sorted.
template <int NT>  // threads per CTA (512 for small k': two CTAs per SM)
__global__ void __launch_bounds__(NT) k_cand_select(const unsigned long long* __restrict__ cand,
                                                      const uint32_t* __restrict__ cand_cnt, uint32_t cand_cap,
                                                      int64_t q0, int kprime, int sort_cap,
                                                      uint32_t* __restrict__ cand_ids,
                                                      float* __restrict__ cand_scores, uint8_t* __restrict__ overflow,
                                                      DevInfo* info, int final_pass,
                                                      const float* __restrict__ theta, GatherDst gd) {
  extern __shared__ unsigned long long sb[];  // sort_cap
  __shared__ uint32_t hist[kHistBins];
  __shared__ uint32_t s_prefix, s_above, s_count, s_ties;
  const int64_t g = blockIdx.x;
  const uint32_t cnt_all = cand_cnt[g];
  uint32_t* oi = cand_ids + (q0 + g) * kprime;
  float* os = cand_scores + (q0 + g) * kprime;
  // shortfall guard: a finite theta_q came from >= k' sampled documents scoring >= theta_q, so the
  // full pass must emit >= k' candidates; fewer means the two passes disagreed on some score (fp32
  // order), and the query is finished on the dense path like an overflow (Alg. 7's V is never short)
  const bool shortfall = theta && theta[g] > -INFINITY && cnt_all < (uint32_t)kprime;
  if (cnt_all > cand_cap || (final_pass && shortfall)) {
    // the row is padded either way: a sample pass then yields no threshold (theta stays); a final
    // pass leaves the query to the dense path (the re-rank that runs before it sees no candidates)
    if (final_pass && threadIdx.x == 0) {
      overflow[q0 + g] = 1;
      atomicAdd(&info->max_id, 1u);  // (search info) number of queries needing the dense path
    }
    for (int t = threadIdx.x; t < kprime; t += blockDim.x) {
      oi[t] = kNoId;
      os[t] = -INFINITY;
      for (int d = 0; d < gd.n; d++) {  // (the dense path rewrites the row at every destination)
        gd.ids[d][gd.off + (q0 + g) * kprime + t] = kNoId;
        gd.scores[d][gd.off + (q0 + g) * kprime + t] = -INFINITY;
      }
    }
    return;
  }
  const unsigned long long* c = cand + g * (int64_t)cand_cap;
  const uint32_t cnt = cnt_all;
  const uint32_t target = min((uint32_t)kprime, cnt);
  int N;
  constexpr uint32_t nt = NT;
  if (cnt > (uint32_t)sort_cap && cnt <= nt * kSelPer) {
    // register radix select: every thread holds up to PER score keys; the key K of the
    // target-th largest is found bit by bit with block-wide counts (no shared-memory atomics)
    if (cnt <= nt * 8) N = reg_select<8, NT>(c, cnt, target, sort_cap, sb, &s_count, &s_ties);
    else if (cnt <= nt * 16) N = reg_select<16, NT>(c, cnt, target, sort_cap, sb, &s_count, &s_ties);
    else N = reg_select<kSelPer, NT>(c, cnt, target, sort_cap, sb, &s_count, &s_ties);
  } else if (cnt <= (uint32_t)sort_cap) {
    N = 1;
    while (N < (int)cnt) N <<= 1;
    for (int t = threadIdx.x; t < N; t += blockDim.x) sb[t] = t < (int)cnt ? c[t] : 0ull;
  } else {
    // exact key K of the target-th largest: three histogram levels over the 32-bit score key
    if (threadIdx.x == 0) {
      s_prefix = 0;
      s_above = 0;
    }
    const int shifts[3] = {20, 8, 0};
    const int widths[3] = {12, 12, 8};
    for (int lv = 0; lv < 3; lv++) {
      for (int b = threadIdx.x; b < kHistBins; b += blockDim.x) hist[b] = 0;
      __syncthreads();
      const int sh = shifts[lv], wd = widths[lv];
      const uint32_t msk = (1u << wd) - 1u;
      const int hs = sh + wd;
      const uint32_t pre = s_prefix;
      for (uint32_t t = threadIdx.x; t < cnt; t += blockDim.x) {
        const uint32_t key = (uint32_t)(c[t] >> 32);
        if (lv > 0 && (key >> hs) != pre) continue;
        atomicAdd(&hist[(key >> sh) & msk], 1u);
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        const uint32_t need = target - s_above;
        uint32_t acc = 0;
        int b = (int)msk;
        for (; b > 0; b--) {
          if (acc + hist[b] >= need) break;
          acc += hist[b];
        }
        s_above += acc;
        s_prefix = (pre << wd) | (uint32_t)b;
      }
      __syncthreads();
    }
    // s_prefix = K; s_above = #keys > K (< target).  When the ties of K do not fit the sort buffer,
    // the (target - above) smallest ids among them are found by the same three histogram levels on
    // the low word ~id (composite order, ties by ascending id), never by atomic arrival order
    const uint32_t K = s_prefix;
    const uint32_t above = s_above;
    __syncthreads();
    uint32_t nt = 0;
    for (uint32_t t = threadIdx.x; t < cnt; t += blockDim.x) nt += (uint32_t)(c[t] >> 32) == K ? 1u : 0u;
    if (threadIdx.x == 0) s_ties = 0;
    __syncthreads();
    nt = __reduce_add_sync(kFull, nt);
    if ((threadIdx.x & 31) == 0 && nt) atomicAdd(&s_ties, nt);
    __syncthreads();
    const uint32_t ties = s_ties;
    uint32_t Lw = 0;
    if (above + ties > (uint32_t)sort_cap) {
      if (threadIdx.x == 0) {
        s_prefix = 0;
        s_above = 0;
      }
      const uint32_t need = target - above;
      for (int lv = 0; lv < 3; lv++) {
        for (int b = threadIdx.x; b < kHistBins; b += blockDim.x) hist[b] = 0;
        __syncthreads();
        const int sh = shifts[lv], wd = widths[lv];
        const uint32_t msk = (1u << wd) - 1u;
        const int hs = sh + wd;
        const uint32_t pre = s_prefix;
        for (uint32_t t = threadIdx.x; t < cnt; t += blockDim.x) {
          const unsigned long long v = c[t];
          if ((uint32_t)(v >> 32) != K) continue;
          const uint32_t lo = (uint32_t)v;
          if (lv > 0 && (lo >> hs) != pre) continue;
          atomicAdd(&hist[(lo >> sh) & msk], 1u);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
          const uint32_t nd = need - s_above;
          uint32_t acc = 0;
          int b = (int)msk;
          for (; b > 0; b--) {
            if (acc + hist[b] >= nd) break;
            acc += hist[b];
          }
          s_above += acc;
          s_prefix = (pre << wd) | (uint32_t)b;
        }
        __syncthreads();
      }
      Lw = s_prefix;
    }
    if (threadIdx.x == 0) s_count = 0;
    __syncthreads();
    for (uint32_t t = threadIdx.x; t < cnt; t += blockDim.x) {
      const unsigned long long v = c[t];
      const uint32_t key = (uint32_t)(v >> 32);
      if (key > K || (key == K && (uint32_t)v >= Lw)) {
        const uint32_t pos = atomicAdd(&s_count, 1u);
        if (pos < (uint32_t)sort_cap) sb[pos] = v;
      }
    }
    __syncthreads();
    const int got = (int)min(s_count, (uint32_t)sort_cap);
    N = 1;
    while (N < got) N <<= 1;
    for (int t = got + threadIdx.x; t < N; t += blockDim.x) sb[t] = 0ull;
  }
  bitonic_desc_u64(sb, N);
  for (int t = threadIdx.x; t < kprime; t += blockDim.x) {
    uint32_t id = kNoId;
    float sc = -INFINITY;
    if (t < (int)target) {
      const unsigned long long v = sb[t];
      id = ~(uint32_t)(v & 0xffffffffu);
      sc = key2f((uint32_t)(v >> 32));
    }
    oi[t] = id;
    os[t] = sc;
    // document shards: the row goes to every shard's gather buffer too (peer stores, coalesced per row)
    for (int d = 0; d < gd.n; d++) {
      gd.ids[d][gd.off + (q0 + g) * kprime + t] = id;
      gd.scores[d][gd.off + (q0 + g) * kprime + t] = sc;
    }
  }
}


int select_sort_cap(int kprime) {
  // room for k' plus ties of the k'-th key
  int p = 1;
  while (p < kprime) p <<= 1;
  return std::min(SINN_MAX_KPRIME, std::max(1024, 2 * p));
}

}  // namespace

bool tile_path_supported(int m, bool lower) { return m <= 512 && warps_per_cta(m, lower) >= 8; }

int tile_qmax() { return kQMax; }

int doc_head_max(int, bool lower, bool) { return doc_head_width(lower); }

int theta_bins() { return kThetaBins; }

void launch_qtab(const int64_t* q_indptr, const int32_t* q_indices, const float* q_values, const int32_t* qlist,
                 int64_t q0, int64_t G, int32_t n, bool upper_only, uint32_t* cnt, uint32_t* qoff, uint32_t* cursor,
                 uint32_t* scan_tmp, uint2* pairs, uint32_t pair_cap, uint32_t* sgn, uint4* dir, const uint16_t* pi,
                 int32_t h, uint32_t* bm, DevInfo* info, cudaStream_t s, int32_t max_terms) {
  cudaMemsetAsync(cnt, 0, sizeof(uint32_t) * (size_t)(n + 1), s);
  if (bm && G <= 1024) cudaMemsetAsync(bm, 0, sizeof(uint32_t) * 32 * (size_t)n, s);
  else {
    bm = nullptr;
    cudaMemsetAsync(cursor, 0, sizeof(uint32_t) * (size_t)n, s);
  }
  if (dir) cudaMemsetAsync(sgn, 0, sizeof(uint32_t) * (size_t)n, s);
  const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((G * 32 + 255) / 256, (int64_t)sm_count() * 8));
  k_qtab_count<<<blocks, 256, 0, s>>>(q_indptr, q_indices, q_values, qlist, q0, G, n, upper_only ? 1 : 0, cnt,
                                      dir ? sgn : nullptr, bm, max_terms, info);
  exclusive_scan_u32(cnt, qoff, n + 1, scan_tmp, s);
  k_qtab_fill<<<blocks, 256, 0, s>>>(q_indptr, q_indices, q_values, qlist, q0, G, n, upper_only ? 1 : 0, qoff, cursor,
                                    pairs, pair_cap, bm, max_terms, info);
  if (dir) {
    const unsigned db = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)sm_count() * 8));
    k_dir_fill<<<db, 256, 0, s>>>(qoff, sgn, pi, pairs, n, h, pair_cap, dir);
  }
}

void launch_doc_score(bool emit, const int64_t* toff, const uint32_t* post, int64_t ntiles_total, int64_t stride,
                      const uint8_t* live, const int32_t* nnz, const void* U, const void* L, bool bf16,
                      const uint16_t* pi, int32_t m, int32_t h, const uint4* dir, const uint2* pairs, int32_t nqc,
                      const float* theta, const uint32_t* list_ok, unsigned long long* cand, uint32_t* cand_cnt,
                      uint32_t cand_cap, uint32_t* hist, uint32_t* nsampled, const float* Qh,
                      const uint32_t* head_cnt, const float* raw_val, const int64_t* raw_off, const uint32_t* allow,
                      int64_t allow_words, uint32_t* sched, cudaStream_t s, QMaskArgs qm, const uint2* cont,
                      const uint8_t* cnum, const int32_t* raw_idx, const int32_t* raw_nnz, float* rows, int64_t skip) {
  DocArgs A{toff, post, (ntiles_total + stride - 1) / stride, stride, live, nnz, U, L, pi, m, h, dir, pairs, nqc,
            theta, list_ok, cand, cand_cnt, cand_cap, hist, nsampled, 1, Qh, head_cnt, raw_val, raw_off, sched,
            allow, allow_words, 0, qm, cont, cnum, raw_idx, raw_nnz, 0};
  A.rows = emit ? nullptr : rows;
  A.skip = emit ? skip : 0;
  // sketch columns by bulk copy + mbarrier (SINN_TMA=1) or cp.async (default: measured 0.4-0.8 % faster,
  // a 0.25-2 KB column is too small for the bulk copy's issue/wait latency to pay)
  if (const char* e = getenv("SINN_TMA")) A.tma = atoi(e) != 0;
  if (bf16) launch_doc_score_bf16(emit, &A, L != nullptr, Qh != nullptr, s);
  else launch_doc_score_tpl<false>(emit, A, L != nullptr, Qh != nullptr, s);
}

// The sampled documents' candidates from the rows the sample pass kept (DocArgs.rows): the full pass
// skips the sampled tiles, and their scores are the very ones theta was derived from.  A warp per
// sampled document; the same admission as k_doc_score's EMIT scan (score >= theta_q, -0.0 == +0.0,
// per-query masks at emission), vacant and batch-masked documents skipped as there.
__global__ void __launch_bounds__(256) k_emit_rows(DocArgs A) {
  const int lane = threadIdx.x & 31;
  const int64_t nd = A.ntiles * kTile;  // sampled document slots
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < nd;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t t = (i / kTile) * A.stride;
    const int d = (int)(i % kTile);
    const uint32_t id = (uint32_t)(t * kTile + d);
    if (!A.live[id]) continue;
    if (A.allow && !(t < A.allow_words && ((__ldg(A.allow + t) >> d) & 1u))) continue;
    const float4* row = reinterpret_cast<const float4*>(A.rows + i * (int64_t)kQMax);
#pragma unroll 2
    for (int k = 0; k < kQMax / 128; k++) {
      const int q0 = 4 * lane + 128 * k;
      if (q0 >= A.nqc) continue;
      const float4 x4 = row[q0 >> 2];
      const float xs[4] = {x4.x, x4.y, x4.z, x4.w};
#pragma unroll
      for (int c = 0; c < 4; c++) {
        const int q = q0 + c;
        if (q >= A.nqc) continue;
        float x = xs[c];
        if (!(x >= __ldg(A.theta + q))) continue;
        if (x == 0.0f) x = 0.0f;  // -0.0 -> +0.0 (R19)
        if (!qmask_pass(A.qm, (uint32_t)q, id)) continue;
        emit(A, (uint32_t)q, x, id);
      }
    }
  }
}

void launch_emit_rows(const float* rows, int64_t ntiles_total, int64_t stride, const uint8_t* live, int32_t nqc,
                      const float* theta, unsigned long long* cand, uint32_t* cand_cnt, uint32_t cand_cap,
                      const uint32_t* allow, int64_t allow_words, QMaskArgs qm, cudaStream_t s) {
  DocArgs A{};
  A.ntiles = (ntiles_total + stride - 1) / stride;
  A.stride = stride;
  A.live = live;
  A.nqc = nqc;
  A.theta = theta;
  A.cand = cand;
  A.cand_cnt = cand_cnt;
  A.cand_cap = cand_cap;
  A.allow = allow;
  A.allow_words = allow_words;
  A.qm = qm;
  A.rows = const_cast<float*>(rows);
  const int64_t warps = A.ntiles * kTile;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((warps + 7) / 8, (int64_t)sm_count() * 32));
  k_emit_rows<<<grid, 256, 0, s>>>(A);
}

// test hook (SINN_TEST_THETA_BUMP=1): theta raised above the sample's bound, so that the full pass
// emits fewer than k' candidates and the shortfall guard of k_cand_select must send the query to the
// dense path (tests/test_gpu_parity.py)
__global__ void k_bump_theta(float* theta, int n) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n && theta[q] > -INFINITY) theta[q] = theta[q] > 0.0f ? theta[q] * 4.0f + 1.0f : 1.0f;
}

// F4: per query of the pass, the live (and batch-allowed) documents of the sampled tiles that pass its
// constraint set — the sample size k_theta compares with k' (warp per query, lane per tile)
__global__ void k_qmask_sampled(const uint8_t* __restrict__ live, const uint32_t* __restrict__ allow,
                                int64_t allow_words, int64_t ntiles, int64_t stride, QMaskArgs qm, int32_t nqc,
                                uint32_t* __restrict__ nsamp_q) {
  const int lane = threadIdx.x & 31;
  const int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (g >= nqc) return;
  const int32_t r = __ldg(qm.qmask + g);
  uint32_t c = 0;
  for (int64_t it = lane; it * stride < ntiles; it += 32) {
    const int64_t t = it * stride;
    uint32_t lw = 0;
    for (int d = 0; d < 32; d++) lw |= (live[t * 32 + d] ? 1u : 0u) << d;
    if (allow) lw &= t < allow_words ? allow[t] : 0u;
    if (r >= 0) lw &= t < qm.words ? __ldg(qm.masks + (int64_t)r * qm.words + t) : 0u;
    c += __popc(lw);
  }
  c = __reduce_add_sync(kFull, c);
  if (lane == 0) nsamp_q[g] = c;
}

void launch_qmask_sampled(const uint8_t* live, const uint32_t* allow, int64_t allow_words, int64_t ntiles,
                          int64_t stride, QMaskArgs qm, int32_t nqc, uint32_t* nsamp_q, cudaStream_t s) {
  k_qmask_sampled<<<(unsigned)((nqc * 32 + 255) / 256), 256, 0, s>>>(live, allow, allow_words, ntiles, stride, qm, nqc,
                                                                   nsamp_q);
}

void launch_theta(const uint32_t* hist, const uint32_t* nsampled, int nqc, int kprime, float* theta,
                  uint32_t* list_ok, cudaStream_t s, const uint32_t* nsamp_q) {
  cudaMemsetAsync(list_ok, 0x01, sizeof(uint32_t), s);
  k_theta<<<(unsigned)nqc, kThetaThreads, 0, s>>>(hist, nsampled, nqc, kprime, theta, list_ok, nsamp_q);
  const char* be = getenv("SINN_TEST_THETA_BUMP");
  const bool bump = be && be[0] == '1';
  if (bump) k_bump_theta<<<(unsigned)((nqc + 255) / 256), 256, 0, s>>>(theta, nqc);
}

void launch_cand_select(const unsigned long long* cand, const uint32_t* cand_cnt, uint32_t cand_cap, int64_t q0,
                        int nqc, int kprime, uint32_t* cand_ids, float* cand_scores, uint8_t* overflow,
                        DevInfo* info, cudaStream_t s, bool final_pass, int64_t expected, const float* theta,
                        const GatherDst* gather) {
  const GatherDst gd = gather ? *gather : GatherDst{};
  smem_optin((const void*)k_cand_select<512>);
  smem_optin((const void*)k_cand_select<1024>);
  const int cap = select_sort_cap(kprime);
  // 512 threads when few candidates are expected (config 2: two CTAs per SM hide the block
  // barriers of the select); their registers hold 16 K keys, so larger candidate sets (config 4 at
  // 4 M documents: ~28 K) keep 1,024 threads
  if (kprime <= 512 && expected >= 0 && expected <= 12288)
    k_cand_select<512><<<(unsigned)nqc, 512, (size_t)cap * 8, s>>>(cand, cand_cnt, cand_cap, q0, kprime, cap,
                                                                   cand_ids, cand_scores, overflow, info,
                                                                   final_pass ? 1 : 0, theta, gd);
  else
    k_cand_select<1024><<<(unsigned)nqc, 1024, (size_t)cap * 8, s>>>(cand, cand_cnt, cand_cap, q0, kprime, cap,
                                                                     cand_ids, cand_scores, overflow, info,
                                                                     final_pass ? 1 : 0, theta, gd);
}

}  // namespace sinn
