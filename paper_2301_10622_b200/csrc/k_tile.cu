// k_tile.cu — the scoring hot path (Alg. 6 + FindLargest k', T = infinity) for a batch of up to
// 1024 queries, organised around 32-document tiles of the tile-major inverted index.
//
//   k_qtab_count/fill  query prep (S0): the batch regrouped term-major — for every term j, the
//                      (query, q_j) pairs with q_j != 0 (q_j > 0 only under Sinnamon+)
//   k_tile_score       persistent, one CTA per SM.  Per tile: the 32 sketch columns are staged
//                      in shared memory, the tile's postings are walked term-major (coalesced
//                      32-bit entries (j << 5) | d), each posting is decoded once per needed sign
//                      from shared memory and accumulated into the on-chip score tile
//                      S[32 docs][1024 queries] (never written to HBM).  Then every query's column
//                      is scanned: HIST mode (sample pass) histograms the scores; EMIT mode keeps
//                      only scores >= theta_q, a provable lower bound on the k'-th largest score.
//   k_theta            theta_q = lower edge of the histogram bin holding the k'-th largest score
//                      of the sample (the k'-th largest of a subset never exceeds that of the set)
//   k_cand_select      exact top-k' of each query's candidates (radix select + bitonic sort)
#include <math.h>

#include <algorithm>

#include "sinn_device.cuh"
#include "sinn_internal.cuh"

namespace sinn {

namespace {

constexpr int kTile = 32;          // documents per tile (entry low 5 bits)
constexpr int kQMax = 1024;        // queries per pass (score tile columns)
constexpr int kTileThreads = 1024;
constexpr int kHistBins = 4096;    // key >> 20
constexpr int kSortCap = SINN_MAX_KPRIME;  // in-smem sort capacity (u64)

// ---------------------------------------------------------------- S0: batch term table
__global__ void k_qtab_count(const int64_t* __restrict__ q_indptr, const int32_t* __restrict__ q_indices,
                             const float* __restrict__ q_values, const int32_t* __restrict__ qlist, int64_t q0,
                             int64_t G, int32_t n, int upper_only, uint32_t* __restrict__ cnt, DevInfo* info) {
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
      atomicAdd(&cnt[j], 1u);
    }
  }
  err = __reduce_or_sync(0xffffffffu, err);
  if (lane == 0 && err) atomicOr(&info->err, err);
}

__global__ void k_qtab_fill(const int64_t* __restrict__ q_indptr, const int32_t* __restrict__ q_indices,
                            const float* __restrict__ q_values, const int32_t* __restrict__ qlist, int64_t q0,
                            int64_t G, int32_t n, int upper_only, const uint32_t* __restrict__ qoff,
                            uint32_t* __restrict__ cursor, uint2* __restrict__ pairs, uint32_t pair_cap,
                            DevInfo* info) {
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
      const uint32_t pos = qoff[j] + atomicAdd(&cursor[j], 1u);
      if (pos < pair_cap) pairs[pos] = make_uint2((uint32_t)g, __float_as_uint(v));
    }
  }
}

// ---------------------------------------------------------------- S1 + S2: tile scoring
enum { kModeHist = 0, kModeEmit = 1 };

struct TileArgs {
  const int64_t* toff;
  const uint32_t* tpost;
  int64_t ntiles;      // tiles visited: t = i * stride, i < ntiles
  int64_t stride;
  const uint8_t* live;
  const float* U;
  const float* L;      // null under Sinnamon+
  const uint16_t* pi;
  int32_t m, h;
  const uint32_t* qoff;
  const uint2* pairs;
  int32_t nqc;         // queries in this pass (<= kQMax)
  const float* theta;  // [nqc]
  unsigned long long* cand;  // [nqc][cand_cap]
  uint32_t* cand_cnt;        // [nqc]
  uint32_t cand_cap;
  uint32_t* hist;            // [nqc][kHistBins]
  uint32_t* zeros;           // [nqc]
};

template <int MODE>
__global__ void __launch_bounds__(kTileThreads, 1) k_tile_score(TileArgs A) {
  extern __shared__ float4 smem4[];
  float* S = reinterpret_cast<float*>(smem4);   // [kTile][kQMax]
  float* skU = S + kTile * kQMax;               // [kTile][m]
  float* skL = skU + kTile * A.m;               // [kTile][m] (unused under Sinnamon+)
  __shared__ uint32_t live_mask;
  const int tid = threadIdx.x;
  const int m = A.m, h = A.h;
  const bool lower = A.L != nullptr;
  for (int i = tid; i < kTile * kQMax; i += kTileThreads) S[i] = 0.0f;
  // the scanning thread of query q = tid keeps theta_q in a register for all tiles
  const float th = (MODE == kModeEmit && tid < A.nqc) ? A.theta[tid] : 0.0f;
  uint32_t zc = 0;
  const int n4 = kTile * m / 4;
  for (int64_t it = blockIdx.x; it < A.ntiles; it += gridDim.x) {
    const int64_t t = it * A.stride;
    // stage the 32 sketch columns (doc-major rows are contiguous: one 128*m-byte block per side)
    {
      const float4* gu = reinterpret_cast<const float4*>(A.U + t * kTile * m);
      float4* su = reinterpret_cast<float4*>(skU);
      for (int k = tid; k < n4; k += kTileThreads) su[k] = __ldg(gu + k);
      if (lower) {
        const float4* gl = reinterpret_cast<const float4*>(A.L + t * kTile * m);
        float4* sl = reinterpret_cast<float4*>(skL);
        for (int k = tid; k < n4; k += kTileThreads) sl[k] = __ldg(gl + k);
      }
      if (tid < 32) {
        const uint32_t mk = __ballot_sync(0xffffffffu, A.live[t * kTile + tid] != 0);
        if (tid == 0) live_mask = mk;
      }
    }
    __syncthreads();
    // postings walk (Alg. 6 lines 4-12 for the batch): entry (j << 5) | d
    const int64_t pb = A.toff[t], pe = A.toff[t + 1];
    for (int64_t p = pb + tid; p < pe; p += kTileThreads) {
      const uint32_t ent = __ldg(A.tpost + p);
      const uint32_t j = ent >> 5, d = ent & 31u;
      const uint32_t qb = __ldg(A.qoff + j), qe = __ldg(A.qoff + j + 1);
      if (qb == qe) continue;
      int cells[SINN_MAX_H];
      for (int o = 0; o < h; o++) cells[o] = __ldg(A.pi + (int64_t)j * h + o);
      float eu = 0.0f, el = 0.0f;
      bool hu = false, hl = false;
      for (uint32_t r = qb; r < qe; r++) {
        const uint2 pr = __ldg(A.pairs + r);
        const float v = __uint_as_float(pr.y);
        float est;
        if (v > 0.0f) {
          if (!hu) {
            eu = decode_upper(skU + d * m, cells, h);
            hu = true;
          }
          est = eu;
        } else {
          if (!hl) {
            el = decode_lower(skL + d * m, cells, h);
            hl = true;
          }
          est = el;
        }
        atomicAdd(&S[d * kQMax + pr.x], v * est);
      }
    }
    __syncthreads();
    // scan the score column of query tid, reset it for the next tile
    if (tid < A.nqc) {
      const uint32_t lm = live_mask;
      for (int d = 0; d < kTile; d++) {
        float* cell = &S[d * kQMax + tid];
        const float x = *cell;
        *cell = 0.0f;
        if (!((lm >> d) & 1u)) continue;
        if (MODE == kModeEmit) {
          if (x >= th) {
            const uint32_t pos = atomicAdd(&A.cand_cnt[tid], 1u);
            if (pos < A.cand_cap)
              A.cand[(int64_t)tid * A.cand_cap + pos] =
                  ((unsigned long long)f2key(x) << 32) | (unsigned long long)(0xffffffffu - (uint32_t)(t * kTile + d));
          }
        } else {
          if (x == 0.0f) zc++;
          else atomicAdd(&A.hist[(int64_t)tid * kHistBins + (f2key(x) >> 20)], 1u);
        }
      }
    }
    __syncthreads();
  }
  if (MODE == kModeHist && tid < A.nqc && zc) atomicAdd(&A.zeros[tid], zc);
}

// ---------------------------------------------------------------- theta
// one warp per query: bin of the k'-th largest sample score -> its lower edge (provable bound)
__global__ void k_theta(const uint32_t* __restrict__ hist, const uint32_t* __restrict__ zeros, int nqc, int kprime,
                        float* __restrict__ theta) {
  const int lane = threadIdx.x & 31;
  const int q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (q >= nqc) return;
  const uint32_t* hq = hist + (int64_t)q * kHistBins;
  constexpr int per = kHistBins / 32;  // lane L owns bins [4096 - (L+1)*per, 4096 - L*per)
  const int top = kHistBins - lane * per;
  const int zbin = (int)(f2key(0.0f) >> 20);
  uint32_t mine = 0;
  for (int b = top - per; b < top; b++) mine += hq[b] + (b == zbin ? zeros[q] : 0u);
  uint32_t inc = mine;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t t = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += t;
  }
  const uint32_t total = __shfl_sync(0xffffffffu, inc, 31);
  if (total < (uint32_t)kprime) {
    if (lane == 0) theta[q] = -INFINITY;  // the sample cannot bound k': every live document is a candidate
    return;
  }
  const uint32_t exc = inc - mine;
  const bool hit = exc < (uint32_t)kprime && inc >= (uint32_t)kprime;
  const int src = __ffs(__ballot_sync(0xffffffffu, hit)) - 1;
  if (lane == src) {
    uint32_t acc = exc;
    int b = top - 1;
    for (; b >= top - per; b--) {
      acc += hq[b] + (b == zbin ? zeros[q] : 0u);
      if (acc >= (uint32_t)kprime) break;
    }
    theta[q] = key2f((uint32_t)b << 20);
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

// one CTA per query.  cnt <= kSortCap: sort everything; otherwise radix-select the score key in
// three levels (12/12/8 bits) until the candidates above the threshold fit the sort buffer.
__global__ void __launch_bounds__(1024) k_cand_select(const unsigned long long* __restrict__ cand,
                                                      const uint32_t* __restrict__ cand_cnt, uint32_t cand_cap,
                                                      int64_t q0, int kprime, uint32_t* __restrict__ cand_ids,
                                                      float* __restrict__ cand_scores, uint8_t* __restrict__ overflow,
                                                      DevInfo* info) {
  extern __shared__ unsigned long long sb[];  // kSortCap
  __shared__ uint32_t hist[kHistBins];
  __shared__ uint32_t s_count, s_prefix, s_above, s_exact, s_need, s_taken;
  __shared__ int s_shift;
  const int64_t g = blockIdx.x;
  const uint32_t cnt_all = cand_cnt[g];
  uint32_t* oi = cand_ids + (q0 + g) * kprime;
  float* os = cand_scores + (q0 + g) * kprime;
  if (cnt_all > cand_cap) {  // candidate buffer overflowed: the dense path finishes this query
    if (threadIdx.x == 0) {
      overflow[q0 + g] = 1;
      atomicAdd(&info->max_id, 1u);  // (search info) number of queries needing the dense path
    }
    return;
  }
  const unsigned long long* c = cand + g * (int64_t)cand_cap;
  const uint32_t cnt = cnt_all;
  const uint32_t target = min((uint32_t)kprime, cnt);
  int N;
  if (cnt <= (uint32_t)kSortCap) {
    N = 1;
    while (N < (int)cnt) N <<= 1;
    for (int t = threadIdx.x; t < N; t += blockDim.x) sb[t] = t < (int)cnt ? c[t] : 0ull;
  } else {
    // radix select on the 32-bit score key (candidate high word)
    if (threadIdx.x == 0) {
      s_prefix = 0;
      s_above = 0;
      s_exact = 0;
      s_shift = 32;
    }
    __syncthreads();
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
        for (; b >= 0; b--) {
          if (acc + hist[b] >= need) break;
          acc += hist[b];
        }
        const uint32_t above = s_above + acc;
        s_prefix = (pre << wd) | (uint32_t)b;
        s_shift = sh;
        if (above + hist[b] <= (uint32_t)kSortCap) {
          s_exact = 0;
          s_above = above;
          s_need = 0xffffffffu;  // resolved: take every key with (key >> sh) >= prefix
        } else if (lv == 2) {
          s_exact = 1;
          s_above = above;
          s_need = target - above;
        } else {
          s_above = above;
          s_need = 0;  // refine
        }
      }
      __syncthreads();
      if (s_need != 0) break;
    }
    if (threadIdx.x == 0) {
      s_count = 0;
      s_taken = 0;
    }
    __syncthreads();
    const uint32_t pre = s_prefix, sh = (uint32_t)s_shift;
    for (uint32_t t = threadIdx.x; t < cnt; t += blockDim.x) {
      const unsigned long long v = c[t];
      const uint32_t key = (uint32_t)(v >> 32);
      bool take;
      if (!s_exact) take = (key >> sh) >= pre;
      else take = key > pre || (key == pre && atomicAdd(&s_taken, 1u) < s_need);
      if (take) {
        const uint32_t pos = atomicAdd(&s_count, 1u);
        if (pos < (uint32_t)kSortCap) sb[pos] = v;
      }
    }
    __syncthreads();
    const int got = (int)min(s_count, (uint32_t)kSortCap);
    N = 1;
    while (N < got) N <<= 1;
    for (int t = got + threadIdx.x; t < N; t += blockDim.x) sb[t] = 0ull;
  }
  bitonic_desc_u64(sb, N);
  for (int t = threadIdx.x; t < kprime; t += blockDim.x) {
    if (t < (int)target) {
      const unsigned long long v = sb[t];
      oi[t] = 0xffffffffu - (uint32_t)(v & 0xffffffffu);
      os[t] = key2f((uint32_t)(v >> 32));
    } else {
      oi[t] = kNoId;
      os[t] = -INFINITY;
    }
  }
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

}  // namespace

size_t tile_smem_bytes(int m, bool lower) {
  return sizeof(float) * ((size_t)kTile * kQMax + (size_t)kTile * m * (lower ? 2 : 1));
}

bool tile_path_supported(int m, bool lower) { return tile_smem_bytes(m, lower) <= 200 * 1024; }

int tile_qmax() { return kQMax; }

void launch_qtab(const int64_t* q_indptr, const int32_t* q_indices, const float* q_values, const int32_t* qlist,
                 int64_t q0, int64_t G, int32_t n, bool upper_only, uint32_t* cnt, uint32_t* qoff, uint32_t* cursor,
                 uint32_t* scan_tmp, uint2* pairs, uint32_t pair_cap, DevInfo* info, cudaStream_t s) {
  cudaMemsetAsync(cnt, 0, sizeof(uint32_t) * (size_t)(n + 1), s);
  cudaMemsetAsync(cursor, 0, sizeof(uint32_t) * (size_t)n, s);
  const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((G * 32 + 255) / 256, 148 * 8));
  k_qtab_count<<<blocks, 256, 0, s>>>(q_indptr, q_indices, q_values, qlist, q0, G, n, upper_only ? 1 : 0, cnt, info);
  exclusive_scan_u32(cnt, qoff, n + 1, scan_tmp, s);
  k_qtab_fill<<<blocks, 256, 0, s>>>(q_indptr, q_indices, q_values, qlist, q0, G, n, upper_only ? 1 : 0, qoff, cursor,
                                    pairs, pair_cap, info);
}

void launch_tile_score(bool emit, const int64_t* toff, const uint32_t* tpost, int64_t ntiles_total, int64_t stride,
                       const uint8_t* live, const float* U, const float* L, const uint16_t* pi, int32_t m, int32_t h,
                       const uint32_t* qoff, const uint2* pairs, int32_t nqc, const float* theta,
                       unsigned long long* cand, uint32_t* cand_cnt, uint32_t cand_cap, uint32_t* hist,
                       uint32_t* zeros, cudaStream_t s) {
  TileArgs A{toff, tpost, (ntiles_total + stride - 1) / stride, stride, live, U, L, pi, m, h, qoff, pairs, nqc,
             theta, cand, cand_cnt, cand_cap, hist, zeros};
  const size_t smem = tile_smem_bytes(m, L != nullptr);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_tile_score<kModeHist>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
    cudaFuncSetAttribute(k_tile_score<kModeEmit>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
    attr = true;
  }
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(num_sms(), A.ntiles));
  if (emit) k_tile_score<kModeEmit><<<grid, kTileThreads, smem, s>>>(A);
  else k_tile_score<kModeHist><<<grid, kTileThreads, smem, s>>>(A);
}

void launch_theta(const uint32_t* hist, const uint32_t* zeros, int nqc, int kprime, float* theta, cudaStream_t s) {
  k_theta<<<(unsigned)((nqc * 32 + 255) / 256), 256, 0, s>>>(hist, zeros, nqc, kprime, theta);
}

void launch_cand_select(const unsigned long long* cand, const uint32_t* cand_cnt, uint32_t cand_cap, int64_t q0,
                        int nqc, int kprime, uint32_t* cand_ids, float* cand_scores, uint8_t* overflow,
                        DevInfo* info, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_cand_select, cudaFuncAttributeMaxDynamicSharedMemorySize, kSortCap * 8);
    attr = true;
  }
  k_cand_select<<<(unsigned)nqc, 1024, kSortCap * 8, s>>>(cand, cand_cnt, cand_cap, q0, kprime, cand_ids, cand_scores,
                                                         overflow, info);
}

}  // namespace sinn
