// k_search.cu — batched search orchestration (Alg. 6 scoring + Alg. 7 ranking, T = infinity).
//
// Main path (k_tile.cu): query prep -> sample pass (histograms) -> theta -> tile scoring pass with
// fused threshold select -> exact top-k' of the candidates.  Dense path (this file), used when a
// query's candidate buffer overflows, when the sketch tile does not fit shared memory, or when
// forced (SINN_FORCE_DENSE=1, for testing): score rows S[G][stride] fp32 in HBM, the same
// tile-major postings walk with red.add into the rows, radix select of the k' largest per row.
// Then for the whole batch:
//   k_rerank        warp per candidate: exact <q, x_v> from the raw-vector store (Alg. 7 l.2-4)
//   k_final         bitonic sort of the k' exact scores -> top-k (Alg. 7 line 5)
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>

#include "sinn_device.cuh"
#include "sinn_internal.cuh"

namespace sinn {

namespace {

constexpr int kCandCap = SINN_MAX_KPRIME;  // candidate buffer per row (u64 composite keys)
constexpr int kBins = 2048;
constexpr int kTieSlices = 4096;  // max slices (blocks) per row of the selection kernels

struct SelState {
  uint32_t prefix;    // key bits fixed so far (right-aligned)
  uint32_t level;     // 1..3: next histogram level; 4 = resolved
  uint32_t mode;      // 0 refine, 1 collect key >= thr, 2 collect key > thr + ties == thr, 3 nothing
  uint32_t thr;       // threshold key
  uint32_t target;    // min(k', non-vacant count)
  uint32_t above;     // elements known to be strictly above the current prefix range
  uint32_t tie_need;  // mode 2: how many key == thr to take
  uint32_t count;     // candidates collected
  uint32_t tie_taken;
  uint32_t pad[3];
};

// level l: bits [shift_lo, shift_lo + width) are histogrammed among keys whose higher bits == prefix
__host__ __device__ inline int level_shift(int l) { return l == 1 ? 21 : (l == 2 ? 10 : 0); }
__host__ __device__ inline int level_width(int l) { return l == 3 ? 10 : 11; }

__device__ __forceinline__ bool col_ok(const uint8_t* live, const uint32_t* allow, int64_t allow_words, int64_t i) {
  return live[i] && (!allow || ((i >> 5) < allow_words && ((allow[i >> 5] >> (i & 31)) & 1u)));
}

__global__ void k_init_scores(float* __restrict__ S, int64_t stride, int64_t cap, const uint8_t* __restrict__ live,
                              const uint32_t* __restrict__ allow, int64_t allow_words, QMaskArgs qm,
                              const int32_t* __restrict__ qlist) {
  float4* row = reinterpret_cast<float4*>(S + (int64_t)blockIdx.y * stride);
  // F4: this row's query constraint set (-1: none)
  const int32_t r = qm.qmask ? __ldg(qm.qmask + qlist[blockIdx.y]) : -1;
  const uint32_t* qw = r >= 0 ? qm.masks + (int64_t)r * qm.words : nullptr;
  auto ok = [&](int64_t i) {
    return i < cap && col_ok(live, allow, allow_words, i) &&
           (!qw || ((i >> 5) < qm.words && ((__ldg(qw + (i >> 5)) >> (i & 31)) & 1u)));
  };
  const int64_t n4 = stride >> 2;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n4; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t << 2;
    float4 v;
    v.x = ok(i + 0) ? 0.0f : -INFINITY;
    v.y = ok(i + 1) ? 0.0f : -INFINITY;
    v.z = ok(i + 2) ? 0.0f : -INFINITY;
    v.w = ok(i + 3) ? 0.0f : -INFINITY;
    row[t] = v;
  }
}

// ---------------------------------------------------------------- dense-path scoring (Alg. 6)
// block per tile: the same tile-major postings walk as the tile kernel, decoding from the HBM
// sketch and accumulating with red.add into the score rows of the queries in the term table.
template <class T>  // sketch cell: float, or bfloat16 bits (F3)
__global__ void __launch_bounds__(256) k_dense_score(const int64_t* __restrict__ toff, const int32_t* __restrict__ tsz,
                                                     const uint32_t* __restrict__ tpost,
                                                     int64_t ntiles, const uint32_t* __restrict__ qoff,
                                                     const uint2* __restrict__ pairs, const T* __restrict__ U,
                                                     const T* __restrict__ L, const uint16_t* __restrict__ pi,
                                                     int32_t m, int32_t h, float* __restrict__ S, int64_t stride,
                                                     const int64_t* __restrict__ raw_off,
                                                     const int32_t* __restrict__ raw_nnz,
                                                     const int32_t* __restrict__ raw_idx,
                                                     const float* __restrict__ raw_val, const uint2* __restrict__ cont,
                                                     const uint8_t* __restrict__ cnum) {
  // one posting (term j, document id): decode and add q_j * estimate to the rows of j's queries
  auto posting = [&](uint32_t j, int64_t id) {
    const uint32_t qb = qoff[j], qe = qoff[j + 1];
    if (qb == qe) return;
    int cells[SINN_MAX_H];
    for (int o = 0; o < h; o++) cells[o] = pi[(int64_t)j * h + o];
    float eu = 0.0f, el = 0.0f;
    bool hu = false, hl = false;
    if (raw_val) {  // exact mode: the stored value (binary search of j in the document's row)
      const int32_t* ri = raw_idx + raw_off[id];
      int32_t lo = 0, hi = raw_nnz[id];
      while (lo < hi) {
        const int32_t mid = (lo + hi) >> 1;
        if (ri[mid] < (int32_t)j) lo = mid + 1; else hi = mid;
      }
      eu = el = raw_val[raw_off[id] + lo];
      hu = hl = true;
    }
    for (uint32_t r = qb; r < qe; r++) {
      const uint2 pr = pairs[r];
      const float v = __uint_as_float(pr.y);
      float est;
      if (v > 0.0f) {
        if (!hu) { eu = decode_upper(U + id * m, cells, h); hu = true; }
        est = eu;
      } else {
        if (!hl) { el = decode_lower(L + id * m, cells, h); hl = true; }
        est = el;
      }
      atomicAdd(&S[(int64_t)pr.x * stride + id], v * est);
    }
  };
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t pb = toff[t], pe = pb + tsz[t];
    for (int64_t p = pb + threadIdx.x; p < pe; p += blockDim.x) {
      const uint32_t ent = tpost[p];
      posting(ent >> 5, t * 32 + (ent & 31u));
    }
    if (cont) {  // bitmap containers (F3): thread = (container, document)
      const int cn = cnum[t];
      for (int k = threadIdx.x; k < cn * 32; k += blockDim.x) {
        const uint2 cv = cont[t * 32 + (k >> 5)];
        if ((cv.y >> (k & 31)) & 1u) posting(cv.x, t * 32 + (k & 31));
      }
    }
  }
}

// ---------------------------------------------------------------- selection (FindLargest k', Alg. 3)
__global__ void k_sel_hist(const float* __restrict__ S, int64_t stride, int64_t len, const SelState* __restrict__ st,
                           int level, uint32_t* __restrict__ hist) {
  const int64_t g = blockIdx.y;
  if (level > 1 && (st[g].mode != 0 || st[g].level != (uint32_t)level)) return;
  __shared__ uint32_t h[kBins];
  for (int t = threadIdx.x; t < kBins; t += blockDim.x) h[t] = 0;
  __syncthreads();
  const int shift = level_shift(level), width = level_width(level);
  const uint32_t mask = (1u << width) - 1u;
  const uint32_t prefix = level > 1 ? st[g].prefix : 0;
  const int hshift = shift + width;
  const int64_t per = ((len + gridDim.x - 1) / gridDim.x + 3) & ~(int64_t)3;
  const int64_t lo = (int64_t)blockIdx.x * per, hi = min(len, lo + per);
  const float* row = S + g * stride;
  for (int64_t i = lo + 4 * (int64_t)threadIdx.x; i < hi; i += 4 * (int64_t)blockDim.x) {
    float4 v4 = *reinterpret_cast<const float4*>(row + i);
    float v[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
    for (int t = 0; t < 4; t++) {
      if (i + t >= hi || v[t] == -INFINITY) continue;
      const uint32_t key = f2key(v[t]);
      if (level > 1 && (hshift >= 32 ? 0u : (key >> hshift)) != prefix) continue;
      atomicAdd(&h[(key >> shift) & mask], 1u);
    }
  }
  __syncthreads();
  uint32_t* gh = hist + g * kBins;
  for (int t = threadIdx.x; t < kBins; t += blockDim.x)
    if (h[t]) atomicAdd(&gh[t], h[t]);
}

// one warp per row: choose the bin holding the target-th largest key
__global__ void k_sel_find(const uint32_t* __restrict__ hist, SelState* __restrict__ st, int64_t G, int level,
                           int kprime) {
  const int lane = threadIdx.x & 31;
  const int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (g >= G) return;
  SelState s = st[g];
  if (level > 1 && (s.mode != 0 || s.level != (uint32_t)level)) return;
  const int width = level_width(level), nb = 1 << width, per = nb / 32;
  const uint32_t* h = hist + g * kBins;
  // lane L owns bins [nb - (L+1)*per, nb - L*per) (top bins first)
  const int top = nb - lane * per;
  uint32_t mine = 0;
  for (int b = top - per; b < top; b++) mine += h[b];
  if (level == 1) {
    uint32_t tot = mine;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, d);
    s.target = min((uint32_t)kprime, tot);
    s.above = 0;
    s.prefix = 0;
    s.count = 0;
    s.tie_taken = 0;
  }
  if (s.target == 0) {
    if (lane == 0) { s.mode = 3; s.level = 4; st[g] = s; }
    return;
  }
  const uint32_t need = s.target - s.above;  // >= 1
  uint32_t inc = mine;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t t = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += t;
  }
  const uint32_t exc = inc - mine;
  const bool hit = exc < need && inc >= need;
  const uint32_t hit_mask = __ballot_sync(0xffffffffu, hit);
  const int src = __ffs(hit_mask) - 1;
  if (lane == src) {
    uint32_t acc = exc;
    int b = top - 1;
    for (; b >= top - per; b--) {
      if (acc + h[b] >= need) break;
      acc += h[b];
    }
    const uint32_t above = s.above + acc;  // strictly above bin b
    const uint32_t inbin = h[b];
    const int shift = level_shift(level);
    const uint32_t prefix = (s.prefix << width) | (uint32_t)b;
    if (above + inbin <= (uint32_t)kCandCap) {
      s.mode = 1;
      s.thr = prefix << shift;
      s.level = 4;
    } else if (level == 3) {
      s.mode = 2;
      s.thr = prefix;  // full 32-bit key
      s.tie_need = s.target - above;
      s.level = 4;
    } else {
      s.mode = 0;
      s.prefix = prefix;
      s.above = above;
      s.level = level + 1;
    }
    st[g] = s;
  }
}

// mode 2 (the ties of the threshold key do not all fit): ties per (row, slice), so that the ties can
// be taken by ascending id — the (score desc, id asc) order of sinn.h / DESIGN.md R10
__global__ void k_sel_tiecount(const float* __restrict__ S, int64_t stride, int64_t len, const SelState* __restrict__ st,
                               uint32_t* __restrict__ tiec) {
  const int64_t g = blockIdx.y;
  if (st[g].mode != 2) return;
  const uint32_t thr = st[g].thr;
  const int64_t per = ((len + gridDim.x - 1) / gridDim.x + 3) & ~(int64_t)3;
  const int64_t lo = (int64_t)blockIdx.x * per, hi = min(len, lo + per);
  const float* row = S + g * stride;
  uint32_t n = 0;
  for (int64_t i = lo + 4 * (int64_t)threadIdx.x; i < hi; i += 4 * (int64_t)blockDim.x) {
    float4 v4 = *reinterpret_cast<const float4*>(row + i);
    float v[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
    for (int t = 0; t < 4; t++)
      if (i + t < hi && v[t] != -INFINITY && f2key(v[t]) == thr) n++;
  }
  n = __reduce_add_sync(0xffffffffu, n);
  if ((threadIdx.x & 31) == 0 && n) atomicAdd(&tiec[g * gridDim.x + blockIdx.x], n);
}

__global__ void __launch_bounds__(256) k_sel_collect(const float* __restrict__ S, int64_t stride, int64_t len,
                                                     SelState* __restrict__ st, unsigned long long* __restrict__ cand,
                                                     const uint32_t* __restrict__ tiec) {
  __shared__ uint32_t wsum[8];
  __shared__ uint32_t s_base;
  const int64_t g = blockIdx.y;
  const uint32_t mode = st[g].mode;
  if (mode == 3) return;
  const uint32_t thr = st[g].thr, tie_need = st[g].tie_need;
  const int64_t per = ((len + gridDim.x - 1) / gridDim.x + 3) & ~(int64_t)3;
  const int64_t lo = (int64_t)blockIdx.x * per, hi = min(len, lo + per);
  const float* row = S + g * stride;
  unsigned long long* out = cand + g * kCandCap;
  // mode 2: rank of this slice's first tie = ties in the slices before it (ascending ids)
  uint32_t rank0 = 0;
  if (mode == 2) {
    if (threadIdx.x == 0) {
      uint32_t b = 0;
      for (unsigned k = 0; k < blockIdx.x; k++) b += tiec[g * gridDim.x + k];
      s_base = b;
    }
    __syncthreads();
    rank0 = s_base;
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int64_t c0 = lo; c0 < hi; c0 += 4 * (int64_t)blockDim.x) {  // (uniform trip count: block scans inside)
    const int64_t i = c0 + 4 * (int64_t)threadIdx.x;
    float v[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
    if (i < hi) {
      float4 v4 = *reinterpret_cast<const float4*>(row + i);
      v[0] = v4.x;
      v[1] = v4.y;
      v[2] = v4.z;
      v[3] = v4.w;
    }
    uint32_t key[4], tie = 0;
#pragma unroll
    for (int t = 0; t < 4; t++) {
      const bool ok = i + t < hi && v[t] != -INFINITY;
      key[t] = ok ? f2key(v[t]) : 0u;
      if (!ok) v[t] = -INFINITY;
      tie |= (mode == 2 && ok && key[t] == thr) ? (1u << t) : 0u;
    }
    uint32_t below = 0;  // ties in this chunk before this thread's (ascending element order)
    if (mode == 2) {
      const uint32_t n = __popc(tie);
      uint32_t inc = n;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += y;
      }
      if (lane == 31) wsum[w] = inc;
      __syncthreads();
      uint32_t wb = 0, tot = 0;
      for (int k = 0; k < nw; k++) {
        wb += k < w ? wsum[k] : 0u;
        tot += wsum[k];
      }
      below = rank0 + wb + inc - n;
      rank0 += tot;
      __syncthreads();
    }
#pragma unroll
    for (int t = 0; t < 4; t++) {
      if (v[t] == -INFINITY) continue;
      bool take;
      if (mode == 1) take = key[t] >= thr;
      else if ((tie >> t) & 1u) take = below++ < tie_need;
      else take = key[t] > thr;
      if (take) {
        const uint32_t pos = atomicAdd(&st[g].count, 1u);
        if (pos < (uint32_t)kCandCap)
          out[pos] = ((unsigned long long)key[t] << 32) | (unsigned long long)(0xffffffffu - (uint32_t)(i + t));
      }
    }
  }
}

// in-smem bitonic sort, descending, of s[0..N) (N power of two)
__device__ void bitonic_desc(unsigned long long* s, int N) {
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

__device__ __forceinline__ int pow2_at_least(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

// one block per row: sort the candidates, emit V (ids, approximate scores), padded
__global__ void k_sel_sort(const SelState* __restrict__ st, const unsigned long long* __restrict__ cand,
                           const int32_t* __restrict__ qlist, int kprime, uint32_t* __restrict__ cand_ids,
                           float* __restrict__ cand_scores, GatherDst gd) {
  extern __shared__ unsigned long long sbuf[];
  const int64_t g = blockIdx.x;
  const SelState s = st[g];
  const int cnt = s.mode == 3 ? 0 : (int)min(s.count, (uint32_t)kCandCap);
  const int N = pow2_at_least(max(cnt, 1));
  for (int t = threadIdx.x; t < N; t += blockDim.x) sbuf[t] = t < cnt ? cand[g * kCandCap + t] : 0ull;
  bitonic_desc(sbuf, N);
  const int take = min((int)s.target, cnt);
  const int64_t qrow = qlist[g];
  uint32_t* oi = cand_ids + qrow * kprime;
  float* os = cand_scores + qrow * kprime;
  for (int t = threadIdx.x; t < kprime; t += blockDim.x) {
    uint32_t id = kNoId;
    float sc = -INFINITY;
    if (t < take) {
      const unsigned long long c = sbuf[t];
      id = 0xffffffffu - (uint32_t)(c & 0xffffffffu);
      sc = key2f((uint32_t)(c >> 32));
    }
    oi[t] = id;
    os[t] = sc;
    for (int d = 0; d < gd.n; d++) {  // document shards: every shard's gather buffer (GatherDst)
      gd.ids[d][gd.off + qrow * kprime + t] = id;
      gd.scores[d][gd.off + qrow * kprime + t] = sc;
    }
  }
}

// ---------------------------------------------------------------- re-rank (Alg. 7 lines 2-4)
// One CTA per query (blockIdx.y) and slice of its candidates.  The query is staged once in a
// shared-memory open-addressing table (term -> q_j); a warp takes one candidate, its lanes walk
// the candidate's stored row (coalesced index loads) and probe the table; the value of an entry
// is loaded only when its term is in the query.  Queries longer than the table fall back to a
// binary search over the query row.  fp32 products summed per lane, then across the warp.
constexpr int kRrSlots = 1024;  // table slots (queries with <= kRrSlots / 2 terms use the table)

__device__ __forceinline__ uint32_t rr_hash(uint32_t j) { return (j * 2654435761u) >> 22; }  // 10 bits

__global__ void __launch_bounds__(256) k_rerank(const int64_t* __restrict__ q_indptr,
                                                const int32_t* __restrict__ q_indices,
                                                const float* __restrict__ q_values, int kprime,
                                                const uint32_t* __restrict__ cand_ids,
                                                const int64_t* __restrict__ raw_off,
                                                const int32_t* __restrict__ raw_nnz,
                                                const int32_t* __restrict__ raw_idx,
                                                const float* __restrict__ raw_val, float* __restrict__ exact,
                                                int64_t g0) {
  __shared__ int32_t tj[kRrSlots];
  __shared__ float tv[kRrSlots];
  const int64_t g = g0 + blockIdx.y;  // (grid.y <= 65,535 per launch: batches are issued in chunks)
  const int lane = threadIdx.x & 31;
  const int warps = blockDim.x >> 5;
  const int64_t qb = q_indptr[g], qn = q_indptr[g + 1] - qb;
  const int32_t* qi = q_indices + qb;
  const float* qv = q_values + qb;
  const bool table = qn <= kRrSlots / 2;
  if (table) {
    for (int t = threadIdx.x; t < kRrSlots; t += blockDim.x) tj[t] = -1;
    __syncthreads();
    for (int64_t p = threadIdx.x; p < qn; p += blockDim.x) {
      const int32_t j = qi[p];
      uint32_t hs = rr_hash((uint32_t)j);
      while (atomicCAS(&tj[hs], -1, j) != -1) hs = (hs + 1) & (kRrSlots - 1);
      tv[hs] = qv[p];
    }
    __syncthreads();
  }
  // a HALF-warp per candidate (two rows in flight per warp: twice the memory-level parallelism of
  // the latency-bound row walk), 16 lanes x 4 row-index loads per step
  const int hl = lane & 15, half = lane >> 4;
  const int hw = 2 * warps;  // half-warps per CTA
  for (int t0 = blockIdx.x * hw + 2 * (threadIdx.x >> 5); t0 < kprime; t0 += gridDim.x * hw) {
    const int t = t0 + half;
    const uint32_t id = t < kprime ? cand_ids[g * kprime + t] : kNoId;
    float acc = 0.0f;
    if (id != kNoId) {
      const int64_t ro = raw_off[id];
      const int32_t rn = raw_nnz[id];
      if (table) {
        // four row-index loads per lane in flight; a value is loaded only for a query term
        for (int32_t p0 = hl; p0 < rn; p0 += 64) {
          int32_t jj[4];
#pragma unroll
          for (int u = 0; u < 4; u++) jj[u] = p0 + 16 * u < rn ? __ldg(raw_idx + ro + p0 + 16 * u) : -1;
#pragma unroll
          for (int u = 0; u < 4; u++) {
            if (jj[u] < 0) continue;
            uint32_t hs = rr_hash((uint32_t)jj[u]);
            int32_t tk;
            while ((tk = tj[hs]) != jj[u] && tk != -1) hs = (hs + 1) & (kRrSlots - 1);
            if (tk == jj[u]) acc = fmaf(tv[hs], __ldg(raw_val + ro + p0 + 16 * u), acc);
          }
        }
      } else {
        for (int32_t p = hl; p < rn; p += 16) {
          const int32_t j = __ldg(raw_idx + ro + p);
          int64_t lo = 0, hi = qn;
          while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (qi[mid] < j) lo = mid + 1; else hi = mid;
          }
          if (lo < qn && qi[lo] == j) acc = fmaf(qv[lo], __ldg(raw_val + ro + p), acc);
        }
      }
    }
#pragma unroll
    for (int d = 8; d > 0; d >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, d);
    if (hl == 0 && t < kprime) exact[g * kprime + t] = id == kNoId ? -INFINITY : acc;
  }
}

// one block per query: top-k of the k' exact (or approximate) scores, ties by ascending id
__global__ void k_final(const uint32_t* __restrict__ cand_ids, const float* __restrict__ scores, int kprime, int k,
                        uint32_t* __restrict__ out_ids, float* __restrict__ out_scores) {
  extern __shared__ unsigned long long sbuf[];
  const int64_t g = blockIdx.x;
  const int N = pow2_at_least(kprime);
  for (int t = threadIdx.x; t < N; t += blockDim.x) {
    unsigned long long c = 0ull;
    if (t < kprime) {
      const uint32_t id = cand_ids[g * kprime + t];
      if (id != kNoId)
        c = ((unsigned long long)f2key(scores[g * kprime + t]) << 32) | (unsigned long long)(0xffffffffu - id);
    }
    sbuf[t] = c;
  }
  bitonic_desc(sbuf, N);
  for (int t = threadIdx.x; t < k; t += blockDim.x) {
    const unsigned long long c = t < N ? sbuf[t] : 0ull;
    if (c != 0ull) {
      out_ids[g * k + t] = 0xffffffffu - (uint32_t)(c & 0xffffffffu);
      out_scores[g * k + t] = key2f((uint32_t)(c >> 32));
    } else {
      out_ids[g * k + t] = kNoId;
      out_scores[g * k + t] = -INFINITY;
    }
  }
}

// one WARP per query for k' <= 32 PER: the k' (score key, ~id) composites sit in registers (PER per
// lane); k rounds of (lane-local max, warp max) take the top-k in order, ties by ascending id — the
// same order as k_final's sort, without its block-wide bitonic network (config 2: 44 -> ~5 us)
template <int PER>
__global__ void __launch_bounds__(256) k_final_warp(const uint32_t* __restrict__ cand_ids,
                                                    const float* __restrict__ scores, int64_t nq, int kprime, int k,
                                                    uint32_t* __restrict__ out_ids, float* __restrict__ out_scores) {
  const int lane = threadIdx.x & 31;
  const int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (g >= nq) return;
  unsigned long long c[PER];
#pragma unroll
  for (int i = 0; i < PER; i++) {
    const int t = i * 32 + lane;
    c[i] = 0ull;
    if (t < kprime) {
      const uint32_t id = cand_ids[g * kprime + t];
      if (id != kNoId)
        c[i] = ((unsigned long long)f2key(scores[g * kprime + t]) << 32) | (unsigned long long)(0xffffffffu - id);
    }
  }
  for (int r = 0; r < k; r++) {
    unsigned long long best = 0ull;
#pragma unroll
    for (int i = 0; i < PER; i++) best = c[i] > best ? c[i] : best;
    unsigned long long wbest = best;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      const unsigned long long o = __shfl_xor_sync(0xffffffffu, wbest, d);
      wbest = o > wbest ? o : wbest;
    }
    if (wbest != 0ull && best == wbest) {  // composites are unique: exactly one lane holds it
#pragma unroll
      for (int i = 0; i < PER; i++)
        if (c[i] == wbest) c[i] = 0ull;
    }
    if (lane == 0) {
      if (wbest != 0ull) {
        out_ids[g * k + r] = 0xffffffffu - (uint32_t)(wbest & 0xffffffffu);
        out_scores[g * k + r] = key2f((uint32_t)(wbest >> 32));
      } else {
        out_ids[g * k + r] = kNoId;
        out_scores[g * k + r] = -INFINITY;
      }
    }
  }
}

// ---------------------------------------------------------------- document sharding
// The path shards by document: shard r of W holds the documents with id % W == r under the local id
// id / W (global = local * W + r).  Per-shard top-k' lists are exchanged once (all-gather), merged
// into the global V by k_merge_topk, re-ranked by their owners (k_owned_local -> k_rerank -> k_final
// -> k_ids_global) and the per-shard top-k merged again.  These kernels are the on-device ends of
// that exchange; the collective itself is NCCL's (torch.distributed).

// merge `parts` lists of kin (id, score) per query into the top-kout by (score desc, global id asc)
struct MergeAdd {
  uint32_t add[kMergeMaxParts];
};
__global__ void k_merge_topk(const uint32_t* __restrict__ ids, const float* __restrict__ scores, int64_t nq, int parts,
                             int kin, uint32_t mul, MergeAdd ad, int kout, uint32_t* __restrict__ out_ids,
                             float* __restrict__ out_scores) {
  extern __shared__ unsigned long long sbuf[];
  const int64_t g = blockIdx.x;
  const int tot = parts * kin;
  const int N = pow2_at_least(tot);
  for (int t = threadIdx.x; t < N; t += blockDim.x) {
    unsigned long long c = 0ull;
    if (t < tot) {
      const int p = t / kin, r = t - p * kin;
      const int64_t at = ((int64_t)p * nq + g) * kin + r;
      const uint32_t id = ids[at];
      if (id != kNoId) {
        const unsigned long long gid = (unsigned long long)id * mul + ad.add[p];
        if (gid < 0xffffffffull)  // (a global id beyond the id range is dropped; documented in sinn.h)
          c = ((unsigned long long)f2key(scores[at] + 0.0f) << 32) | (0xffffffffull - gid);  // (-0.0 ties +0.0)
      }
    }
    sbuf[t] = c;
  }
  bitonic_desc(sbuf, N);
  for (int t = threadIdx.x; t < kout; t += blockDim.x) {
    const unsigned long long c = t < N ? sbuf[t] : 0ull;
    if (c != 0ull) {
      out_ids[g * kout + t] = 0xffffffffu - (uint32_t)(c & 0xffffffffu);
      out_scores[g * kout + t] = key2f((uint32_t)(c >> 32));
    } else {
      out_ids[g * kout + t] = kNoId;
      out_scores[g * kout + t] = -INFINITY;
    }
  }
}

// global candidate ids -> this shard's local ids (kNoId for candidates it does not own or hold live)
__global__ void k_owned_local(const uint32_t* __restrict__ gids, int64_t count, uint32_t mul, uint32_t add,
                              const uint8_t* __restrict__ live, int64_t cap, uint32_t* __restrict__ local) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t g = gids[t];
    uint32_t l = kNoId;
    if (g != kNoId && g >= add && (g - add) % mul == 0) {
      const uint32_t c = (g - add) / mul;
      if ((int64_t)c < cap && live[c]) l = c;
    }
    local[t] = l;
  }
}

// local result ids -> global ids, in place
__global__ void k_ids_global(uint32_t* __restrict__ ids, int64_t count, uint32_t mul, uint32_t add) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t l = ids[t];
    if (l != kNoId) ids[t] = l * mul + add;
  }
}

template <typename T>
T* carve(char*& p, size_t count) {
  T* r = reinterpret_cast<T*>(p);
  p += ((count * sizeof(T) + 255) / 256) * 256;
  return r;
}

size_t align256(size_t b) { return ((b + 255) / 256) * 256; }

}  // namespace

static int64_t score_budget_bytes() {
  static int64_t b = -1;
  if (b < 0) {
    const char* e = getenv("SINN_SCORE_BYTES");
    b = e ? atoll(e) : (int64_t)2 << 30;
    if (b < (1 << 20)) b = 1 << 20;
  }
  return b;
}

static bool force_dense() {
  const char* e = getenv("SINN_FORCE_DENSE");
  return e && e[0] == '1';
}

// Head terms (lists covering most documents, on most queries of a batch) are taken out of the sparse
// walk when some term's list covers >= kHeadDocFrac of the live documents:
//   default        k_doc_score with the per-document dense product of <= 8 head terms (HD)
//   SINN_HEAD=1    the tile kernel k_head_score (k_head.cu; slower as built, profiles/r1_head_*)
//   SINN_HEAD=0    plain sparse walk;  SINN_HEAD=d forces the per-document product
constexpr double kHeadDocFrac = 0.15;
constexpr float kHeadTau = 0.15f;  // min expected fraction of (document, query) pairs a head term touches

static char head_override() {
  const char* e = getenv("SINN_HEAD");
  return e ? e[0] : 'a';
}

static float head_tau() {
  const char* e = getenv("SINN_HEAD_TAU");
  return e ? (float)atof(e) : kHeadTau;
}

// L2 residency control (north star: "L2-residency control for hot sketches"): the batch's term table,
// pairs and directory — read by every scoring warp for every index entry, while the sketch cells and
// ids stream through L2 once — are marked persisting for the call (a stream access-policy window over
// their contiguous carve; the device's persisting set-aside is reserved once).  The caller's window
// is restored on exit.  SINN_L2_PERSIST=0 disables it (A/B).
struct L2Window {
  cudaStream_t s;
  bool on = false;
  cudaStreamAttrValue old{};
  L2Window(cudaStream_t s_, const void* base, size_t bytes) : s(s_) {
    const char* e = getenv("SINN_L2_PERSIST");
    if (e && e[0] == '0') return;
    static int maxw[256] = {}, setaside[256] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 256) return;
    if (!maxw[dev]) {
      cudaDeviceGetAttribute(&maxw[dev], cudaDevAttrMaxAccessPolicyWindowSize, dev);
      int lim = 0;
      cudaDeviceGetAttribute(&lim, cudaDevAttrMaxPersistingL2CacheSize, dev);
      setaside[dev] = std::min(lim, 16 << 20);
      if (setaside[dev] > 0) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)setaside[dev]);
      cudaGetLastError();
    }
    if (maxw[dev] <= 0 || setaside[dev] <= 0 || bytes == 0) return;
    if (cudaStreamGetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &old) != cudaSuccess) {
      cudaGetLastError();
      return;
    }
    cudaStreamAttrValue v{};
    v.accessPolicyWindow.base_ptr = const_cast<void*>(base);
    v.accessPolicyWindow.num_bytes = std::min<size_t>(bytes, (size_t)maxw[dev]);
    v.accessPolicyWindow.hitRatio = std::min(1.0f, (float)setaside[dev] / (float)v.accessPolicyWindow.num_bytes);
    v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    on = cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v) == cudaSuccess;
    cudaGetLastError();
  }
  ~L2Window() {
    if (on) cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &old);
    cudaGetLastError();
  }
};

// grow-only workspace slot (stream-ordered pool allocation, as the index arrays)
static cudaError_t ensure(void** p, size_t* have, size_t need, cudaStream_t s) {
  if (*have >= need) return cudaSuccess;
  if (*p) cudaFreeAsync(*p, s);
  *p = nullptr;
  *have = 0;
  cudaError_t e = cudaMallocAsync(p, need, s);
  if (e == cudaSuccess && getenv("SINN_POISON")) cudaMemsetAsync(*p, 0xA5, need, s);  // (debug: dirty memory)
  if (e == cudaSuccess) *have = need;
  return e;
}

// candidates per query per pass (main path); the sample stride keeps ~cap / 4 expected (held in
// registers by k_cand_select): 112 K rather than 64 K lets configs 3 and 5 sample 1/28 and 1/14 of
// the documents instead of 1/16 and 1/8 (+2.6 % and +4 % QPS at full size)
constexpr uint32_t kTileCandCapDefault = 114688;
static uint32_t tile_cand_cap() {
  const char* e = getenv("SINN_CAND_CAP");
  return e ? (uint32_t)std::max(4096, atoi(e)) : kTileCandCapDefault;
}
constexpr int kHeadRows = 16;  // head-term query rows (Qh) reserved per pass

// Dense path for the queries qlist[0..count) (device list): score rows in HBM + radix select.
static cudaError_t dense_batch(sinn_index* idx, const SearchArgs& a, const int32_t* qlist, int64_t count,
                               cudaStream_t s, std::string* why) {
  const int64_t cap = idx->cap, ntiles = cap / 32, n = idx->n;
  const int64_t stride = std::max<int64_t>(32, ((cap + 31) / 32) * 32);
  int64_t G = score_budget_bytes() / (stride * 4);
  G = std::max<int64_t>(1, std::min<int64_t>(G, count));
  G = std::min<int64_t>(G, 65535);
  const int kp = a.kprime;
  uint32_t pair_cap = (uint32_t)std::min<int64_t>((int64_t)G * n, 0x3fffffffLL);
  size_t need = align256(sizeof(float) * (size_t)(G * stride)) + align256(sizeof(uint32_t) * (size_t)(G * kBins)) +
                align256(sizeof(SelState) * (size_t)G) + align256(sizeof(unsigned long long) * (size_t)(G * kCandCap)) +
                align256(sizeof(uint32_t) * (size_t)(G * kTieSlices)) +
                3 * align256(sizeof(uint32_t) * (size_t)(n + 1)) +
                align256(sizeof(uint32_t) * exclusive_scan_u32_tmp_elems(n + 1)) +
                align256(sizeof(uint2) * (size_t)pair_cap) + 1024;
  cudaError_t e = ensure(&idx->ws3, &idx->ws3_bytes, need, s);
  if (e != cudaSuccess) {
    *why = "dense-path workspace allocation failed";
    return e;
  }
  char* p = static_cast<char*>(idx->ws3);
  float* S = carve<float>(p, (size_t)(G * stride));
  uint32_t* hist = carve<uint32_t>(p, (size_t)(G * kBins));
  SelState* st = carve<SelState>(p, (size_t)G);
  unsigned long long* cand = carve<unsigned long long>(p, (size_t)(G * kCandCap));
  uint32_t* tiec = carve<uint32_t>(p, (size_t)(G * kTieSlices));
  uint32_t* qcnt = carve<uint32_t>(p, (size_t)(n + 1));
  uint32_t* qoff = carve<uint32_t>(p, (size_t)(n + 1));
  uint32_t* cursor = carve<uint32_t>(p, (size_t)(n + 1));
  uint32_t* scan_tmp = carve<uint32_t>(p, exclusive_scan_u32_tmp_elems(n + 1));
  uint2* pairs = carve<uint2>(p, (size_t)pair_cap);
  smem_optin((const void*)k_sel_sort);
  const int64_t len = stride;
  for (int64_t c0 = 0; c0 < count; c0 += G) {
    const int64_t g = std::min<int64_t>(G, count - c0);
    launch_qtab(a.q_indptr, a.q_indices, a.q_values, qlist + c0, 0, g, idx->n, idx->upper_only && !a.exact, qcnt, qoff, cursor,
                scan_tmp, pairs, pair_cap, nullptr, nullptr, idx->pi, idx->h, nullptr, idx->d_sinfo, s, a.max_terms);
    count_launch(idx, SINN_PH_SCORE, 4);
    {
      PhaseScope ps(idx, SINN_PH_INIT, s);
      int bx = (int)std::max<int64_t>(1, std::min<int64_t>((stride / 4 + 255) / 256, ((int64_t)sm_count() * 16 + g - 1) / g));
      QMaskArgs qm{a.qmasks, a.qmask_words, a.nmasks, a.qmask};
      k_init_scores<<<dim3(bx, (unsigned)g), 256, 0, s>>>(S, stride, cap, idx->live, a.allow, a.allow_words, qm,
                                                          qlist + c0);
      count_launch(idx, SINN_PH_INIT);
    }
    if (ntiles > 0 && idx->post_len > 0) {
      PhaseScope ps(idx, SINN_PH_SCORE, s);
      count_launch(idx, SINN_PH_SCORE);
      const unsigned dgrid = (unsigned)std::min<int64_t>(ntiles, (int64_t)sm_count() * 16);
      if (idx->bf16)
        k_dense_score<<<dgrid, 256, 0, s>>>(idx->off, idx->tsz, idx->post, ntiles, qoff, pairs, idx->Ub, idx->Lb, idx->pi,
                                            idx->m, idx->h, S, stride, idx->raw_off, idx->raw_nnz, idx->raw_idx,
                                            a.exact ? idx->raw_val : nullptr, idx->containers ? idx->cont : nullptr,
                                            idx->cnum);
      else
        k_dense_score<<<dgrid, 256, 0, s>>>(idx->off, idx->tsz, idx->post, ntiles, qoff, pairs, idx->U, idx->L, idx->pi,
                                            idx->m, idx->h, S, stride, idx->raw_off, idx->raw_nnz, idx->raw_idx,
                                            a.exact ? idx->raw_val : nullptr, idx->containers ? idx->cont : nullptr,
                                            idx->cnum);
    }
    PhaseScope ps(idx, SINN_PH_SELECT, s);
    count_launch(idx, SINN_PH_SELECT, 9);
    cudaMemsetAsync(hist, 0, sizeof(uint32_t) * (size_t)(g * kBins), s);
    cudaMemsetAsync(st, 0, sizeof(SelState) * (size_t)g, s);
    int slices = (int)std::max<int64_t>(1, std::min<int64_t>((len + 4095) / 4096, ((int64_t)sm_count() * 8 + g - 1) / g));
    slices = std::min(slices, kTieSlices);
    dim3 hgrid(slices, (unsigned)g);
    k_sel_hist<<<hgrid, 256, 0, s>>>(S, stride, len, st, 1, hist);
    k_sel_find<<<(unsigned)((g * 32 + 255) / 256), 256, 0, s>>>(hist, st, g, 1, kp);
    for (int level = 2; level <= 3; level++) {
      cudaMemsetAsync(hist, 0, sizeof(uint32_t) * (size_t)(g * kBins), s);
      k_sel_hist<<<hgrid, 256, 0, s>>>(S, stride, len, st, level, hist);
      k_sel_find<<<(unsigned)((g * 32 + 255) / 256), 256, 0, s>>>(hist, st, g, level, kp);
    }
    cudaMemsetAsync(tiec, 0, sizeof(uint32_t) * (size_t)g * slices, s);
    k_sel_tiecount<<<hgrid, 256, 0, s>>>(S, stride, len, st, tiec);
    k_sel_collect<<<hgrid, 256, 0, s>>>(S, stride, len, st, cand, tiec);
    k_sel_sort<<<(unsigned)g, 1024, kCandCap * 8, s>>>(st, cand, qlist + c0, kp, a.cand_ids, a.cand_scores, a.gather);
  }
  return cudaGetLastError();
}

static cudaError_t rerank_final(sinn_index* idx, const SearchArgs& a, float* exact, cudaStream_t s) {
  const int kp = a.kprime;
  const int64_t nq = a.nq;
  const float* fin = a.cand_scores;
  if (a.rerank) {
    PhaseScope ps(idx, SINN_PH_RERANK, s);
    count_launch(idx, SINN_PH_RERANK);
    int ns = std::max(1, std::min(16, (kp + 63) / 64));
    // grid.y is limited to 65,535: larger batches are re-ranked in chunks of queries
    for (int64_t g0 = 0; g0 < nq; g0 += 65535) {
      dim3 grid(ns, (unsigned)std::min<int64_t>(65535, nq - g0));
      k_rerank<<<grid, 256, 0, s>>>(a.q_indptr, a.q_indices, a.q_values, kp, a.cand_ids, idx->raw_off, idx->raw_nnz,
                                    idx->raw_idx, idx->raw_val, exact, g0);
    }
    fin = exact;
  }
  int N = 1;
  while (N < kp) N <<= 1;
  smem_optin((const void*)k_final);
  PhaseScope ps(idx, SINN_PH_FINAL, s);
  count_launch(idx, SINN_PH_FINAL);
  const unsigned wgrid = (unsigned)((nq * 32 + 255) / 256);
  if (kp <= 32 * 4 && a.k <= 64)
    k_final_warp<4><<<wgrid, 256, 0, s>>>(a.cand_ids, fin, nq, kp, a.k, a.out_ids, a.out_scores);
  else if (kp <= 32 * 16 && a.k <= 64)
    k_final_warp<16><<<wgrid, 256, 0, s>>>(a.cand_ids, fin, nq, kp, a.k, a.out_ids, a.out_scores);
  else if (kp <= 32 * 32 && a.k <= 32)  // (k rounds: the block sort wins for k = 100, config 5)
    k_final_warp<32><<<wgrid, 256, 0, s>>>(a.cand_ids, fin, nq, kp, a.k, a.out_ids, a.out_scores);
  else
    k_final<<<(unsigned)nq, 512, (size_t)N * 8, s>>>(a.cand_ids, fin, kp, a.k, a.out_ids, a.out_scores);
  return cudaGetLastError();
}

// Owner re-rank of caller-supplied GLOBAL candidates (Alg. 7 lines 2-5 on this shard's part of V)
cudaError_t rerank_candidates(sinn_index* idx, int64_t nq, const int64_t* q_indptr, const int32_t* q_indices,
                              const float* q_values, int32_t kc, const uint32_t* cand_gids, uint32_t mul, uint32_t add,
                              int32_t k, uint32_t* out_ids, float* out_scores, cudaStream_t s, std::string* why) {
  const size_t cnt = (size_t)nq * (size_t)kc;
  cudaError_t e = ensure(&idx->ws, &idx->ws_bytes, 2 * align256(sizeof(uint32_t) * cnt) + 1024, s);
  if (e != cudaSuccess) {
    *why = "re-rank workspace allocation failed";
    return e;
  }
  char* p = static_cast<char*>(idx->ws);
  uint32_t* local = carve<uint32_t>(p, cnt);
  float* exact = carve<float>(p, cnt);
  const unsigned grid = (unsigned)std::min<int64_t>(((int64_t)cnt + 255) / 256, (int64_t)sm_count() * 16);
  count_launch(idx, SINN_PH_RERANK, 2);
  k_owned_local<<<grid, 256, 0, s>>>(cand_gids, (int64_t)cnt, mul, add, idx->live, idx->cap, local);
  SearchArgs a{nq, q_indptr, q_indices, q_values, k, kc, true, out_ids, out_scores, local, nullptr};
  e = rerank_final(idx, a, exact, s);
  if (e != cudaSuccess) return e;
  const int64_t oc = nq * (int64_t)k;
  k_ids_global<<<(unsigned)std::min<int64_t>((oc + 255) / 256, (int64_t)sm_count() * 16), 256, 0, s>>>(out_ids, oc, mul, add);
  return cudaGetLastError();
}

cudaError_t launch_merge_topk(int64_t nq, int32_t parts, int32_t kin, const uint32_t* ids, const float* scores,
                              uint32_t mul, const uint32_t* add, int32_t kout, uint32_t* out_ids, float* out_scores,
                              cudaStream_t s) {
  MergeAdd ad{};
  for (int p = 0; p < parts; p++) ad.add[p] = add ? add[p] : 0u;
  int N = 1;
  while (N < parts * kin) N <<= 1;
  smem_optin((const void*)k_merge_topk);
  // (grid.x up to 2^31 - 1: one CTA per query)
  k_merge_topk<<<(unsigned)nq, N >= 4096 ? 1024 : (N >= 512 ? 512 : 128), (size_t)N * 8, s>>>(
      ids, scores, nq, parts, kin, mul, ad, kout, out_ids, out_scores);
  return cudaGetLastError();
}

cudaError_t search_batch(sinn_index* idx, const SearchArgs& a_in, bool sync, cudaStream_t s, std::string* why,
                         bool* needs_retry) {
  SearchArgs a = a_in;
  *needs_retry = false;
  const int64_t nq = a.nq;
  if (nq == 0) return cudaSuccess;
  const int64_t cap = idx->cap, ntiles = cap / 32, n = idx->n;
  const int kp = a.kprime;
  const int QM = tile_qmax();
  // exact mode always uses k_doc_score (it needs no sketch tile); its overflow fallback is the dense
  // path of the approximate scores, so exact searches are issued with k' large enough (sinn_search_exact)
  const bool tile_ok = a.exact || (tile_path_supported(idx->m, !idx->upper_only) && !force_dense());
  const char hov = head_override();
  const bool has_head = idx->live_count > 0 && idx->max_df >= kHeadDocFrac * (double)idx->live_count;
  const bool doc_head = tile_ok && !a.exact && (hov == 'd' || (hov == 'a' && has_head));
  const bool qtab_upper = idx->upper_only && !a.exact;  // exact MIPS keeps negative query values
  const uint32_t kTileCandCap = tile_cand_cap();
  const uint32_t cand_cap = kTileCandCap;
  // sample stride: a sample of >= 64 k' documents (so that, with sparse queries, enough sampled
  // documents have non-zero scores to bound the k'-th), and few enough candidates (~k' x stride);
  // without head terms (sparse score rows: the sample pass is cheap per document) a sample twice
  // as large halves the candidates (config 2: -2.6% per batch; with head terms, where every
  // sampled cell is histogrammed, the larger sample costs more than it saves)
  const int64_t live_docs = std::max<int64_t>(idx->live_count, 1);
  const int64_t sample_x = getenv("SINN_SAMPLE_X") ? std::max(1, atoi(getenv("SINN_SAMPLE_X")))
                                                   : (has_head ? 64 : 128);
  int64_t stride = std::min<int64_t>(live_docs / (sample_x * (int64_t)kp), (int64_t)kTileCandCap / (4 * (int64_t)kp));
  stride = std::max<int64_t>(1, stride);
  // with dense score rows (head terms) every sampled cell costs a histogram atomic: a nested
  // sample 8x smaller first gives theta_1 (a provable bound of the k'-th largest of the small
  // sample, hence <= that of the large one, which contains it); the large sample then
  // histograms only cells >= theta_1 when theta_1 > 0 (the cells below, zeros included, lie
  // below its k'-th largest), and its k'-th largest is theta
  const char* ce = getenv("SINN_CASCADE");
  const bool cascade = tile_ok && (ce ? atoi(ce) != 0 : (has_head && stride >= 8 && !a.exact));
  // the large sample keeps its documents' score rows, and the full pass skips the sampled tiles: their
  // candidates come from the kept rows (k_emit_rows) — 1 / stride of the full pass for a row write and
  // read (config 5: stride 14).  SINN_ROWS=0 disables it (A/B).
  const char* re_ = getenv("SINN_ROWS");
  const bool keep_rows = cascade && stride > 1 && !a.exact && (re_ ? atoi(re_) != 0 : true);
  const int64_t row_slots = keep_rows ? ((ntiles + stride - 1) / stride) * 32 : 0;
  if (tile_ok && !a.exact) {
    idx->last_stride = stride;
    idx->last_rows = keep_rows ? 1 : 0;
  }
  // ---- workspace (ws): candidates, overflow flags, term table, tile-pass buffers
  const int64_t G = std::min<int64_t>(QM, nq);
  if (idx->pair_cap < (uint32_t)(G * 256)) idx->pair_cap = (uint32_t)(G * 256);
  const uint32_t pair_cap = idx->pair_cap;
  size_t need = 3 * align256(sizeof(uint32_t) * (size_t)(nq * kp)) + align256((size_t)nq) +
                align256(sizeof(int32_t) * (size_t)nq) + 3 * align256(sizeof(uint32_t) * (size_t)(n + 1)) +
                align256(sizeof(uint32_t) * exclusive_scan_u32_tmp_elems(n + 1)) +
                align256(sizeof(uint2) * (size_t)pair_cap) + 4 * align256(sizeof(float) * (size_t)QM) +
                align256(sizeof(uint32_t) * (size_t)QM * theta_bins()) + align256(sizeof(uint32_t) * (size_t)n) +
                align256(2 * sizeof(uint4) * (size_t)n) + 2 * align256(sizeof(uint32_t)) +
                align256(sizeof(uint32_t) * 32 * (size_t)n);
  if (tile_ok) need += align256(sizeof(unsigned long long) * (size_t)G * cand_cap);
  const bool hbuf = doc_head;
  if (hbuf)
    need += align256(sizeof(float) * (size_t)kHeadRows * QM) + 2 * align256(sizeof(uint32_t)) +
            align256(sizeof(unsigned long long) * (size_t)head_cand_cap());
  need += align256(sizeof(float) * (size_t)row_slots * (size_t)QM);
  need += 4096;
  cudaError_t e = ensure(&idx->ws, &idx->ws_bytes, need, s);
  if (e != cudaSuccess) {
    *why = "search workspace allocation failed";
    return e;
  }
  char* p = static_cast<char*>(idx->ws);
  uint32_t* cand_ids_ws = carve<uint32_t>(p, (size_t)(nq * kp));
  float* cand_scores_ws = carve<float>(p, (size_t)(nq * kp));
  float* exact = carve<float>(p, (size_t)(nq * kp));
  uint8_t* overflow = carve<uint8_t>(p, (size_t)nq);
  int32_t* qlist = carve<int32_t>(p, (size_t)nq);
  uint32_t* qcnt = carve<uint32_t>(p, (size_t)(n + 1));
  uint32_t* qoff = carve<uint32_t>(p, (size_t)(n + 1));
  uint32_t* cursor = carve<uint32_t>(p, (size_t)(n + 1));
  uint32_t* scan_tmp = carve<uint32_t>(p, exclusive_scan_u32_tmp_elems(n + 1));
  // the per-batch structures every scoring warp reads (term table, directory) are carved next to each
  // other so one L2 persisting window covers them
  uint2* pairs = carve<uint2>(p, (size_t)pair_cap);
  uint4* dir = carve<uint4>(p, 2 * (size_t)n);
  float* theta = carve<float>(p, (size_t)QM);
  uint32_t* zeros = carve<uint32_t>(p, (size_t)QM);
  uint32_t* nsamp_q = carve<uint32_t>(p, (size_t)QM);  // F4: per-query sample sizes
  uint32_t* ccnt = carve<uint32_t>(p, (size_t)QM);
  uint32_t* hist = carve<uint32_t>(p, (size_t)QM * theta_bins());
  uint32_t* sgn = carve<uint32_t>(p, (size_t)n);
  uint32_t* list_ok = carve<uint32_t>(p, 1);
  uint32_t* sched = carve<uint32_t>(p, 1);  // k_doc_score's work-unit counter
  uint32_t* qbm = carve<uint32_t>(p, 32 * (size_t)n);  // per-term query bitmaps of a 1024-query chunk
  unsigned long long* cand = tile_ok ? carve<unsigned long long>(p, (size_t)G * cand_cap) : nullptr;
  float* Qh = hbuf ? carve<float>(p, (size_t)kHeadRows * QM) : nullptr;
  uint32_t* head_cnt = hbuf ? carve<uint32_t>(p, 1) : nullptr;
  uint32_t* nhcand = hbuf ? carve<uint32_t>(p, 1) : nullptr;
  unsigned long long* hcand = hbuf ? carve<unsigned long long>(p, (size_t)head_cand_cap()) : nullptr;
  float* rows = row_slots ? carve<float>(p, (size_t)row_slots * (size_t)QM) : nullptr;
  if (!a.cand_ids) {
    a.cand_ids = cand_ids_ws;
    a.cand_scores = cand_scores_ws;
  }
  cudaMemsetAsync(overflow, 0, (size_t)nq, s);
  L2Window l2w(s, qoff, (const char*)(dir + 2 * (size_t)n) - (const char*)qoff);

  if (tile_ok) {
    const int QC = QM;  // queries per pass
    for (int64_t q0 = 0; q0 < nq; q0 += QC) {
      const int64_t g = std::min<int64_t>(QC, nq - q0);
      const float* th_used = nullptr;  // theta of the sample pass (the shortfall guard's reference)
      const QMaskArgs qmp{a.qmasks, a.qmask_words, a.nmasks, a.qmask ? a.qmask + q0 : nullptr};  // F4, this pass
      {
        PhaseScope ps(idx, SINN_PH_PREP, s);
        count_launch(idx, SINN_PH_PREP, 5);
        launch_qtab(a.q_indptr, a.q_indices, a.q_values, nullptr, q0, g, idx->n, qtab_upper, qcnt, qoff,
                    cursor, scan_tmp, pairs, pair_cap, sgn, dir, idx->pi, idx->h, qbm, idx->d_sinfo, s, a.max_terms);
      }
      if (ntiles > 0 && idx->live_count > 0) {
        cudaMemsetAsync(hist, 0, sizeof(uint32_t) * (size_t)g * theta_bins(), s);
        cudaMemsetAsync(zeros, 0, sizeof(uint32_t), s);  // zeros[0]: live documents in the sample
        cudaMemsetAsync(ccnt, 0, sizeof(uint32_t) * (size_t)g, s);
        const float* dQh = nullptr;
        if (doc_head) {  // head terms of this batch -> per-document dense product inside k_doc_score
          PhaseScope ps(idx, SINN_PH_PREP, s);
          count_launch(idx, SINN_PH_PREP, 2);
          launch_head_select(qoff, idx->df, idx->n, idx->live_count, g, head_tau(), pairs, dir, Qh, head_cnt, hcand,
                             nhcand, doc_head_max(idx->m, !idx->upper_only), QM, s);
          dQh = Qh;
        }
        {
          PhaseScope ps(idx, SINN_PH_INIT, s);  // sample pass + theta
          auto sample = [&](int64_t st, const float* floor_, float* keep = nullptr) {
            launch_doc_score(false, idx->off, idx->post, ntiles, st, idx->live, idx->ecnt, idx->sU(),
                             idx->upper_only ? nullptr : idx->sL(), idx->bf16, idx->pi, idx->m, idx->h, dir, pairs,
                             (int)g, floor_, list_ok, cand, ccnt, kTileCandCap, hist, zeros, dQh, head_cnt,
                             a.exact ? idx->raw_val : nullptr, idx->raw_off, a.allow, a.allow_words, sched, s, qmp,
                             idx->containers ? idx->cont : nullptr, idx->cnum, idx->raw_idx, idx->raw_nnz, keep);
            if (qmp.qmask)
              launch_qmask_sampled(idx->live, a.allow, a.allow_words, ntiles, st, qmp, (int)g, nsamp_q, s);
            launch_theta(hist, zeros, (int)g, kp, theta, list_ok, s, qmp.qmask ? nsamp_q : nullptr);
          };
          if (cascade) {  // (nested sample: see `cascade` above)
            count_launch(idx, SINN_PH_INIT, 4);
            sample(stride * 8, nullptr);
            cudaMemsetAsync(hist, 0, sizeof(uint32_t) * (size_t)g * theta_bins(), s);
            cudaMemsetAsync(zeros, 0, sizeof(uint32_t), s);
            sample(stride, theta, rows);
          } else {
            count_launch(idx, SINN_PH_INIT, 2);
            sample(stride, nullptr);
          }
        }
        th_used = theta;
        {
          PhaseScope ps(idx, SINN_PH_SCORE, s);
          count_launch(idx, SINN_PH_SCORE);
          launch_doc_score(true, idx->off, idx->post, ntiles, 1, idx->live, idx->ecnt, idx->sU(),
                           idx->upper_only ? nullptr : idx->sL(), idx->bf16, idx->pi, idx->m, idx->h, dir, pairs, (int)g, theta,
                           list_ok, cand, ccnt, kTileCandCap, hist, zeros, dQh, head_cnt,
                           a.exact ? idx->raw_val : nullptr, idx->raw_off, a.allow,
                           a.allow_words, sched, s, qmp, idx->containers ? idx->cont : nullptr, idx->cnum,
                           idx->raw_idx, idx->raw_nnz, nullptr, rows ? stride : 0);
          if (rows) {  // the sampled tiles' candidates, from the rows the sample pass kept
            count_launch(idx, SINN_PH_SCORE);
            launch_emit_rows(rows, ntiles, stride, idx->live, (int)g, theta, cand, ccnt, kTileCandCap, a.allow,
                             a.allow_words, qmp, s);
          }
        }
      } else {
        cudaMemsetAsync(ccnt, 0, sizeof(uint32_t) * (size_t)g, s);
      }
      PhaseScope ps(idx, SINN_PH_SELECT, s);
      count_launch(idx, SINN_PH_SELECT);
      launch_cand_select(cand, ccnt, cand_cap, q0, (int)g, kp, a.cand_ids, a.cand_scores, overflow,
                         idx->d_sinfo, s, true, (int64_t)kp * stride, th_used, &a.gather);
    }
  } else {
    // every query takes the dense path
    std::vector<int32_t> all(nq);
    for (int64_t q = 0; q < nq; q++) all[q] = (int32_t)q;
    cudaMemcpyAsync(qlist, all.data(), sizeof(int32_t) * (size_t)nq, cudaMemcpyHostToDevice, s);
    e = dense_batch(idx, a, qlist, nq, s, why);
    if (e != cudaSuccess) return e;
    cudaStreamSynchronize(s);  // `all` must outlive the copy
  }
  if (a.out_ids) {
    e = rerank_final(idx, a, exact, s);
    if (e != cudaSuccess) return e;
  }
  e = cudaGetLastError();
  if (e != cudaSuccess || !tile_ok) return e;
  if (!sync) return cudaSuccess;
  // ---- synchronous completion: term-table overflow -> retry; candidate overflow -> dense path
  e = cudaMemcpyAsync(idx->h_info, idx->d_sinfo, sizeof(DevInfo), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return e;
  const DevInfo inf = *idx->h_info;
  if (inf.err) return cudaSuccess;  // invalid input: the caller reports SINN_EINVAL
  if (inf.pad) {                    // the term table was too small for this batch: grow and redo
    idx->pair_cap = std::max<uint32_t>(idx->pair_cap * 2, (uint32_t)std::min<int64_t>(G * n, 0x3fffffffLL));
    *needs_retry = true;
    return cudaSuccess;
  }
  if (inf.max_id == 0) return cudaSuccess;
  std::vector<uint8_t> fl(nq);
  e = cudaMemcpy(fl.data(), overflow, (size_t)nq, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return e;
  std::vector<int32_t> lst;
  for (int64_t q = 0; q < nq; q++)
    if (fl[q]) lst.push_back((int32_t)q);
  e = cudaMemcpyAsync(qlist, lst.data(), sizeof(int32_t) * lst.size(), cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return e;
  e = dense_batch(idx, a, qlist, (int64_t)lst.size(), s, why);
  if (e != cudaSuccess) return e;
  if (a.out_ids) e = rerank_final(idx, a, exact, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  return e;
}

}  // namespace sinn
