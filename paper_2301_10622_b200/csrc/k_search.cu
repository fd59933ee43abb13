// k_search.cu — batched search (Alg. 6 scoring + Alg. 7 ranking, T = infinity).
//
// Per chunk of G queries (score rows S[G][stride] fp32 in a device workspace):
//   k_init_scores   S[g][i] = 0 for live i, -inf for vacant ("scores[i] <- 0 for all i")
//   k_score         query-batched postings walk: CTA (slice s, query g) walks slice s of every
//                   inverted list I[j], j in nz(q_g); coalesced id loads; decode = min over the h
//                   U cells (q_j > 0) or max over the L cells (q_j < 0); red.add q_j * e into S
//   k_sel_hist/find radix select of the k' largest per row (11/11/10-bit levels; a level is read
//                   only for rows whose candidate bin would overflow the candidate buffer)
//   k_sel_collect   candidates (key >= threshold, exact ties counted) -> per-row buffer
//   k_sel_sort      bitonic sort of the candidates (score desc, id asc) -> V (Alg. 7 line 1)
// Then for the whole batch:
//   k_rerank        warp per candidate: exact <q, x_v> from the raw-vector store (Alg. 7 l.2-4)
//   k_final         bitonic sort of the k' exact scores -> top-k (Alg. 7 line 5)
#include <math.h>

#include <algorithm>

#include "sinn_device.cuh"
#include "sinn_internal.cuh"

namespace sinn {

namespace {

constexpr int kCandCap = SINN_MAX_KPRIME;  // candidate buffer per row (u64 composite keys)
constexpr int kBins = 2048;

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

__global__ void k_init_scores(float* __restrict__ S, int64_t stride, int64_t cap, const uint8_t* __restrict__ live) {
  float4* row = reinterpret_cast<float4*>(S + (int64_t)blockIdx.y * stride);
  const int64_t n4 = stride >> 2;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n4; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t << 2;
    float4 v;
    v.x = (i + 0 < cap && live[i + 0]) ? 0.0f : -INFINITY;
    v.y = (i + 1 < cap && live[i + 1]) ? 0.0f : -INFINITY;
    v.z = (i + 2 < cap && live[i + 2]) ? 0.0f : -INFINITY;
    v.w = (i + 3 < cap && live[i + 3]) ? 0.0f : -INFINITY;
    row[t] = v;
  }
}

// ---------------------------------------------------------------- scoring (Alg. 6)
__global__ void __launch_bounds__(256) k_score(const int64_t* __restrict__ q_indptr, const int32_t* __restrict__ q_indices,
                                               const float* __restrict__ q_values, int64_t q0, int32_t n,
                                               const int64_t* __restrict__ off, const uint32_t* __restrict__ post,
                                               const float* __restrict__ U, const float* __restrict__ L,
                                               const uint16_t* __restrict__ pi, int32_t m, int32_t h, int upper_only,
                                               float* __restrict__ S, int64_t stride, DevInfo* info) {
  const int64_t g = blockIdx.y;
  const int s = blockIdx.x, ns = gridDim.x;
  const int64_t qb = q_indptr[q0 + g], qe = q_indptr[q0 + g + 1];
  float* __restrict__ Sg = S + g * stride;
  if (s == 0 && threadIdx.x == 0 && qe < qb) atomicOr(&info->err, kErrIndptr);
  for (int64_t e = qb; e < qe; e++) {
    const int32_t j = q_indices[e];
    const float q = q_values[e];
    const bool bad = j < 0 || j >= n || !isfinite(q) || (e > qb && q_indices[e - 1] >= j);
    if (bad) {
      if (s == 0 && threadIdx.x == 0) atomicOr(&info->err, kErrRow);
      continue;
    }
    if (q == 0.0f) continue;                 // nz(q)
    const bool positive = q > 0.0f;
    if (!positive && upper_only) continue;   // Sinnamon+: 0 lower-bounds x >= 0 (R6)
    int cells[SINN_MAX_H];
    for (int o = 0; o < h; o++) cells[o] = pi[(int64_t)j * h + o];
    const float* __restrict__ sk = positive ? U : L;
    const int64_t b = off[j], len = off[j + 1] - b;
    const int64_t lo = b + len * s / ns, hi = b + len * (s + 1) / ns;
    for (int64_t p = lo + threadIdx.x; p < hi; p += blockDim.x) {
      const uint32_t i = post[p];
      const float* col = sk + (int64_t)i * m;
      const float est = positive ? decode_upper(col, cells, h) : decode_lower(col, cells, h);
      atomicAdd(&Sg[i], q * est);
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

__global__ void k_sel_collect(const float* __restrict__ S, int64_t stride, int64_t len, SelState* __restrict__ st,
                              unsigned long long* __restrict__ cand) {
  const int64_t g = blockIdx.y;
  const uint32_t mode = st[g].mode;
  if (mode == 3) return;
  const uint32_t thr = st[g].thr, tie_need = st[g].tie_need;
  const int64_t per = ((len + gridDim.x - 1) / gridDim.x + 3) & ~(int64_t)3;
  const int64_t lo = (int64_t)blockIdx.x * per, hi = min(len, lo + per);
  const float* row = S + g * stride;
  unsigned long long* out = cand + g * kCandCap;
  for (int64_t i = lo + 4 * (int64_t)threadIdx.x; i < hi; i += 4 * (int64_t)blockDim.x) {
    float4 v4 = *reinterpret_cast<const float4*>(row + i);
    float v[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
    for (int t = 0; t < 4; t++) {
      if (i + t >= hi || v[t] == -INFINITY) continue;
      const uint32_t key = f2key(v[t]);
      bool take;
      if (mode == 1) take = key >= thr;
      else take = key > thr || (key == thr && atomicAdd(&st[g].tie_taken, 1u) < tie_need);
      if (take) {
        const uint32_t pos = atomicAdd(&st[g].count, 1u);
        if (pos < (uint32_t)kCandCap)
          out[pos] = ((unsigned long long)key << 32) | (unsigned long long)(0xffffffffu - (uint32_t)(i + t));
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
__global__ void k_sel_sort(const SelState* __restrict__ st, const unsigned long long* __restrict__ cand, int64_t q0,
                           int kprime, uint32_t* __restrict__ cand_ids, float* __restrict__ cand_scores) {
  extern __shared__ unsigned long long sbuf[];
  const int64_t g = blockIdx.x;
  const SelState s = st[g];
  const int cnt = s.mode == 3 ? 0 : (int)min(s.count, (uint32_t)kCandCap);
  const int N = pow2_at_least(max(cnt, 1));
  for (int t = threadIdx.x; t < N; t += blockDim.x) sbuf[t] = t < cnt ? cand[g * kCandCap + t] : 0ull;
  bitonic_desc(sbuf, N);
  const int take = min((int)s.target, cnt);
  uint32_t* oi = cand_ids + (q0 + g) * kprime;
  float* os = cand_scores + (q0 + g) * kprime;
  for (int t = threadIdx.x; t < kprime; t += blockDim.x) {
    if (t < take) {
      const unsigned long long c = sbuf[t];
      oi[t] = 0xffffffffu - (uint32_t)(c & 0xffffffffu);
      os[t] = key2f((uint32_t)(c >> 32));
    } else {
      oi[t] = kNoId;
      os[t] = -INFINITY;
    }
  }
}

// ---------------------------------------------------------------- re-rank (Alg. 7 lines 2-4)
__global__ void __launch_bounds__(256) k_rerank(const int64_t* __restrict__ q_indptr,
                                                const int32_t* __restrict__ q_indices,
                                                const float* __restrict__ q_values, int kprime,
                                                const uint32_t* __restrict__ cand_ids,
                                                const int64_t* __restrict__ raw_off,
                                                const int32_t* __restrict__ raw_nnz,
                                                const int32_t* __restrict__ raw_idx,
                                                const float* __restrict__ raw_val, float* __restrict__ exact) {
  const int64_t g = blockIdx.y;
  const int lane = threadIdx.x & 31;
  const int warps = blockDim.x >> 5;
  const int64_t qb = q_indptr[g], qn = q_indptr[g + 1] - qb;
  const int32_t* qi = q_indices + qb;
  const float* qv = q_values + qb;
  for (int t = blockIdx.x * warps + (threadIdx.x >> 5); t < kprime; t += gridDim.x * warps) {
    const uint32_t id = cand_ids[g * kprime + t];
    float acc = 0.0f;
    if (id != kNoId) {
      const int64_t ro = raw_off[id];
      const int32_t rn = raw_nnz[id];
      for (int32_t p = lane; p < rn; p += 32) {
        const int32_t j = raw_idx[ro + p];
        int64_t lo = 0, hi = qn;
        while (lo < hi) {
          const int64_t mid = (lo + hi) >> 1;
          if (qi[mid] < j) lo = mid + 1; else hi = mid;
        }
        if (lo < qn && qi[lo] == j) acc = fmaf(qv[lo], raw_val[ro + p], acc);
      }
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, d);
    if (lane == 0) exact[g * kprime + t] = id == kNoId ? -INFINITY : acc;
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

cudaError_t search_batch(sinn_index* idx, const SearchArgs& a, cudaStream_t s, std::string* why) {
  const int64_t nq = a.nq;
  if (nq == 0) return cudaSuccess;
  const int64_t cap = idx->cap;
  const int64_t stride = std::max<int64_t>(32, ((cap + 31) / 32) * 32);
  int64_t G = score_budget_bytes() / (stride * 4);
  G = std::max<int64_t>(1, std::min<int64_t>(G, nq));
  G = std::min<int64_t>(G, 65535);
  const int kp = a.kprime;

  // workspace
  size_t need = align256(sizeof(float) * (size_t)(G * stride)) + align256(sizeof(uint32_t) * (size_t)(G * kBins)) +
                align256(sizeof(SelState) * (size_t)G) + align256(sizeof(unsigned long long) * (size_t)(G * kCandCap)) +
                2 * align256(sizeof(uint32_t) * (size_t)(nq * kp)) + align256(sizeof(float) * (size_t)(nq * kp)) + 1024;
  if (idx->ws_bytes < need) {
    if (idx->ws) cudaFree(idx->ws);
    idx->ws = nullptr;
    idx->ws_bytes = 0;
    cudaError_t e = cudaMalloc(&idx->ws, need);
    if (e != cudaSuccess) {
      *why = "search workspace allocation failed";
      return e;
    }
    idx->ws_bytes = need;
  }
  char* p = static_cast<char*>(idx->ws);
  float* S = carve<float>(p, (size_t)(G * stride));
  uint32_t* hist = carve<uint32_t>(p, (size_t)(G * kBins));
  SelState* st = carve<SelState>(p, (size_t)G);
  unsigned long long* cand = carve<unsigned long long>(p, (size_t)(G * kCandCap));
  uint32_t* cand_ids = a.cand_ids ? a.cand_ids : carve<uint32_t>(p, (size_t)(nq * kp));
  float* cand_scores = a.cand_scores ? a.cand_scores : carve<float>(p, (size_t)(nq * kp));
  float* exact = carve<float>(p, (size_t)(nq * kp));

  static bool attrs = false;
  if (!attrs) {
    cudaFuncSetAttribute(k_sel_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, kCandCap * 8);
    cudaFuncSetAttribute(k_final, cudaFuncAttributeMaxDynamicSharedMemorySize, kCandCap * 8);
    attrs = true;
  }

  const int64_t len = stride;  // rows are scanned over the full (padded, -inf) stride
  for (int64_t q0 = 0; q0 < nq; q0 += G) {
    const int64_t g = std::min<int64_t>(G, nq - q0);
    {
      PhaseScope ps(idx, SINN_PH_INIT, s);
      int bx = (int)std::max<int64_t>(1, std::min<int64_t>((stride / 4 + 255) / 256, (148 * 16 + g - 1) / g));
      k_init_scores<<<dim3(bx, (unsigned)g), 256, 0, s>>>(S, stride, cap, idx->live);
      count_launch(idx, SINN_PH_INIT);
    }
    {
    PhaseScope ps(idx, SINN_PH_SCORE, s);
    count_launch(idx, SINN_PH_SCORE);
    if (cap > 0 && idx->post_len > 0) {
      // slices per query: enough CTAs to fill the GPU several times over
      int ns = (int)std::max<int64_t>(1, std::min<int64_t>(64, (148 * 8 + g - 1) / g));
      dim3 grid(ns, (unsigned)g);
      k_score<<<grid, 256, 0, s>>>(a.q_indptr, a.q_indices, a.q_values, q0, idx->n, idx->off, idx->post, idx->U,
                                   idx->L, idx->pi, idx->m, idx->h, idx->upper_only ? 1 : 0, S, stride, idx->d_sinfo);
    } else {
      // still validate the query rows
      dim3 grid(1, (unsigned)g);
      k_score<<<grid, 32, 0, s>>>(a.q_indptr, a.q_indices, a.q_values, q0, idx->n, idx->off, idx->post, idx->U,
                                  idx->L, idx->pi, idx->m, idx->h, idx->upper_only ? 1 : 0, S, stride, idx->d_sinfo);
    }
    }
    PhaseScope ps(idx, SINN_PH_SELECT, s);
    count_launch(idx, SINN_PH_SELECT, 8);
    cudaMemsetAsync(hist, 0, sizeof(uint32_t) * (size_t)(g * kBins), s);
    cudaMemsetAsync(st, 0, sizeof(SelState) * (size_t)g, s);
    int slices = (int)std::max<int64_t>(1, std::min<int64_t>((len + 4095) / 4096, (148 * 8 + g - 1) / g));
    dim3 hgrid(slices, (unsigned)g);
    k_sel_hist<<<hgrid, 256, 0, s>>>(S, stride, len, st, 1, hist);
    k_sel_find<<<(unsigned)((g * 32 + 255) / 256), 256, 0, s>>>(hist, st, g, 1, kp);
    for (int level = 2; level <= 3; level++) {
      cudaMemsetAsync(hist, 0, sizeof(uint32_t) * (size_t)(g * kBins), s);
      k_sel_hist<<<hgrid, 256, 0, s>>>(S, stride, len, st, level, hist);
      k_sel_find<<<(unsigned)((g * 32 + 255) / 256), 256, 0, s>>>(hist, st, g, level, kp);
    }
    k_sel_collect<<<hgrid, 256, 0, s>>>(S, stride, len, st, cand);
    k_sel_sort<<<(unsigned)g, 1024, kCandCap * 8, s>>>(st, cand, q0, kp, cand_ids, cand_scores);
  }
  if (a.out_ids) {
    const float* fin = cand_scores;
    if (a.rerank) {
      PhaseScope ps(idx, SINN_PH_RERANK, s);
      count_launch(idx, SINN_PH_RERANK);
      int ns = std::max(1, std::min(64, (kp + 7) / 8));
      dim3 grid(ns, (unsigned)nq);
      k_rerank<<<grid, 256, 0, s>>>(a.q_indptr, a.q_indices, a.q_values, kp, cand_ids, idx->raw_off, idx->raw_nnz,
                                    idx->raw_idx, idx->raw_val, exact);
      fin = exact;
    }
    int N = 1;
    while (N < kp) N <<= 1;
    PhaseScope ps(idx, SINN_PH_FINAL, s);
    count_launch(idx, SINN_PH_FINAL);
    k_final<<<(unsigned)nq, 1024, (size_t)N * 8, s>>>(cand_ids, fin, kp, a.k, a.out_ids, a.out_scores);
  }
  return cudaGetLastError();
}

}  // namespace sinn
