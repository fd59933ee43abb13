// k_head.cu — dense-head split of the scoring path (Alg. 6) for skewed (Zipf) workloads.
//
// In configs 3 and 5 a few coordinates occur in most documents and most queries: their lists make
// up most of Alg. 6's updates (SURVEY.md §7 hard part 2, Appendix A).  For those "head" terms the
// update set  S[d][q] += q_j * e_dj  is a dense product over a tile of 32 documents,
//   S_tile[32 x 1024] += E[32 x H] . Q[H x 1024],
// done here with register-tiled FP32 FFMA (no tensor cores: BASELINE.json; fp32 parity).  Every
// other ("tail") entry takes the sparse per-document walk of k_tile.cu's kernel.  The scores are
// the same sums (Alg. 6) in another order.
//
//   k_head_cand / k_head_pick  per batch: terms with df[j]/live * (queries of j)/nq >= tau (the
//                              expected fraction of (document, query) pairs the term touches),
//                              the best kHMax of them; builds Q[H][1024] (q_j, 0 if absent) and
//                              marks the terms in the batch directory (no sparse pairs)
//   k_head_score               persistent CTA of 1024 threads per SM; per 32-document tile:
//                              warp w walks document w: head entries write E+[hh][w] (upper-bound
//                              decode) and E-[hh][w] (lower), tail entries add into the shared
//                              score row S[w][*]; then thread q (= query q) forms
//                              S[d][q] + sum_hh q_hh * E(sign q_hh)[hh][d] for the 32 documents in
//                              registers (E rows are warp-broadcast shared loads), compares with
//                              theta_q and emits candidates.
//   k_theta_from_sel           theta_q from a sample pass: the k'-th largest sampled score
#include <math.h>

#include <algorithm>

#include "sinn_device.cuh"
#include "sinn_internal.cuh"

namespace sinn {

namespace {

constexpr int kHQ = 512;             // queries per head pass (a 1,024-query batch takes two)
constexpr int kHDocs = 64;           // documents per CTA tile (two index tiles)
constexpr int kHMax = 16;            // head terms per batch
constexpr int kHeadCandCap = 4096;   // head candidates considered
constexpr int kNarrowMax = 8;        // tail terms with more queries are walked warp-cooperatively
constexpr uint32_t kFull = 0xffffffffu;
constexpr uint32_t kHeadMark = 0x80000000u;


__global__ void k_head_cand(const uint32_t* __restrict__ qoff, const int32_t* __restrict__ df, int32_t n,
                            float inv_live, float inv_nq, float tau, unsigned long long* __restrict__ cand,
                            uint32_t* __restrict__ ncand) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t qc = qoff[j + 1] - qoff[j];
    if (qc == 0) continue;
    const float cover = (float)df[j] * inv_live * ((float)qc * inv_nq);
    if (cover >= tau) {
      const uint32_t pos = atomicAdd(ncand, 1u);
      if (pos < (uint32_t)kHeadCandCap)
        cand[pos] = ((unsigned long long)__float_as_uint(cover) << 32) | (unsigned long long)(~(uint32_t)j);
    }
  }
}

// one block: the kHMax best candidates (coverage desc, term asc) -> head list, Q rows, directory marks
__global__ void __launch_bounds__(1024) k_head_pick(const unsigned long long* __restrict__ cand,
                                                    const uint32_t* __restrict__ ncand,
                                                    const uint32_t* __restrict__ qoff, const uint2* __restrict__ pairs,
                                                    uint4* __restrict__ dir, float* __restrict__ Qh,
                                                    uint32_t* __restrict__ head_cnt, int hmax, int qrow) {
  __shared__ unsigned long long sb[kHeadCandCap];
  __shared__ uint32_t hj[kHMax];
  const uint32_t cnt = min(*ncand, (uint32_t)kHeadCandCap);
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
  const int hc = (int)min(cnt, (uint32_t)hmax);
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
    uint4 a = dir[2 * (int64_t)j];
    a.y = (a.y & 0xc0000000u) | a.x;  // no sparse pairs: the term is in the dense product
    dir[2 * (int64_t)j] = a;
    uint4 b = dir[2 * (int64_t)j + 1];
    b.x = kHeadMark | threadIdx.x;  // no inline pairs for a head term (its pair range is empty)
    dir[2 * (int64_t)j + 1] = b;
  }
  if (threadIdx.x == 0) *head_cnt = (uint32_t)hc;
}

__device__ __forceinline__ void emit_h(unsigned long long* cand, uint32_t* cand_cnt, uint32_t cap, uint32_t q, float x,
                                       uint32_t id) {
  const uint32_t pos = atomicAdd(&cand_cnt[q], 1u);
  if (pos < cap) cand[(int64_t)q * cap + pos] = ((unsigned long long)f2key(x) << 32) | (unsigned long long)(~id);
}

struct HeadArgs {
  const int64_t* toff;
  const uint32_t* post;
  int64_t ntiles32;  // index tiles (32 documents)
  int64_t nvisit;    // CTA tiles (64 documents) visited: T = it * stride
  int64_t stride;
  const uint8_t* live;
  const int32_t* nnz;
  const float* U;
  const float* L;
  const uint16_t* pi;
  int32_t m, h;
  const uint4* dir;
  const uint2* pairs;
  int32_t nqc;  // queries of this pass (<= kHQ)
  const float* theta;
  const float* Qh;  // [kHMax][kHQ]
  const uint32_t* head_cnt;
  unsigned long long* cand;
  uint32_t* cand_cnt;
  uint32_t cand_cap;
};

// shared memory: S [64 docs][kHQ] | E+ [kHMax][64] | E- [kHMax][64] | tags [32 warps][kHQ] u8 |
// sketch column per warp (m or 2m) | LPT assignment [64] u8
__host__ __device__ inline size_t head_smem_bytes(int m, bool lower) {
  return sizeof(float) * ((size_t)kHDocs * kHQ + 2 * (size_t)kHMax * kHDocs) + (size_t)32 * kHQ +
         sizeof(float) * (size_t)32 * m * (lower ? 2 : 1) + 64;
}

template <bool LOWER>
struct HeadTail {
  // one 32-entry chunk of a document's index entries: term, directory sector
  uint32_t j;
  uint4 a, b;
};

template <int H, bool LOWER>
__device__ __forceinline__ HeadTail<LOWER> head_load(const HeadArgs& A, int64_t eb, uint32_t p0, uint32_t cnt,
                                                      int lane) {
  HeadTail<LOWER> c;
  const uint32_t p = p0 + lane;
  c.j = p < cnt ? (__ldg(A.post + eb + p) >> 5) : 0xffffffffu;
  c.a = make_uint4(0, 0, 0, 0);
  c.b = make_uint4(0, 0, 0, 0);
  if (c.j != 0xffffffffu) {
    c.a = __ldg(A.dir + 2 * (int64_t)c.j);
    c.b = __ldg(A.dir + 2 * (int64_t)c.j + 1);
  }
  return c;
}

// Persistent CTA of 1024 threads per SM; a CTA tile is 64 documents (two index tiles) x 512 queries.
// Phase 1: warp w walks the two documents the LPT assignment gave it (longest with shortest), head
// entries -> E+/E-[hh][doc], tail entries -> shared row S[doc][*].  Phase 2: thread (half, q) owns
// query q for the 32 documents of its half: S + sum_hh q_hh * E[hh][doc] in registers, compare with
// theta_q, emit.
template <int H, bool LOWER>
__global__ void __launch_bounds__(1024, 1) k_head_score(HeadArgs A) {
  extern __shared__ float4 smem4[];
  float* S = reinterpret_cast<float*>(smem4);  // [64][kHQ]
  float* Ep = S + kHDocs * kHQ;                // [kHMax][64]
  float* Em = Ep + kHMax * kHDocs;             // [kHMax][64]
  uint8_t* tags = reinterpret_cast<uint8_t*>(Em + kHMax * kHDocs);  // [32][kHQ]
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int m = A.m, h = H > 0 ? H : A.h;
  float* colU = reinterpret_cast<float*>(tags + 32 * kHQ) + (size_t)w * m * (LOWER ? 2 : 1);
  float* colL = colU + m;
  uint8_t* asg = reinterpret_cast<uint8_t*>(reinterpret_cast<float*>(tags + 32 * kHQ) + (size_t)32 * m * (LOWER ? 2 : 1));
  uint8_t* tag = tags + w * kHQ;
  const int half = t >> 9, q = t & (kHQ - 1);
  const int nqc = A.nqc;
  const bool qok = q < nqc;
  const float th = qok ? A.theta[q] : INFINITY;
  const int hc = (int)*A.head_cnt;
  float v[kHMax];
#pragma unroll
  for (int hh = 0; hh < kHMax; hh++) v[hh] = (hh < hc && qok) ? A.Qh[hh * kHQ + q] : 0.0f;
#pragma unroll
  for (int d = 0; d < 32; d++) S[(32 * half + d) * kHQ + q] = 0.0f;
  __syncthreads();
  for (int64_t it = blockIdx.x; it < A.nvisit; it += gridDim.x) {
    const int64_t T = it * A.stride;
    // the two index tiles of this CTA tile: per-document entry counts and offsets (every warp)
    uint32_t c_l[2], st_l[2], lm[2];
    int64_t tb[2];
#pragma unroll
    for (int k = 0; k < 2; k++) {
      const int64_t t32 = 2 * T + k;
      const bool ok = t32 < A.ntiles32;
      const int64_t i = t32 * 32 + lane;
      const bool lv = ok && A.live[i] != 0;
      c_l[k] = lv ? (uint32_t)A.nnz[i] : 0u;
      uint32_t inc = c_l[k];
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, inc, d);
        if (lane >= d) inc += y;
      }
      st_l[k] = inc - c_l[k];
      lm[k] = __ballot_sync(kFull, lv);
      tb[k] = ok ? A.toff[t32] : 0;
    }
    if (w == 0) {
      // LPT pairing: rank the 64 documents by entry count (ties by index), pair rank r with 63 - r
      const uint32_t ka = (c_l[0] << 7) | (uint32_t)lane, kb = (c_l[1] << 7) | (uint32_t)(32 + lane);
      uint32_t ra = 0, rb = 0;
      for (int s2 = 0; s2 < 32; s2++) {
        const uint32_t xa = __shfl_sync(kFull, ka, s2), xb = __shfl_sync(kFull, kb, s2);
        ra += (xa > ka) + (xb > ka);
        rb += (xa > kb) + (xb > kb);
      }
      asg[ra < 32 ? 2 * ra : 2 * (63 - ra) + 1] = (uint8_t)lane;
      asg[rb < 32 ? 2 * rb : 2 * (63 - rb) + 1] = (uint8_t)(32 + lane);
    }
    for (int k2 = t; k2 < 2 * kHMax * kHDocs; k2 += blockDim.x) Ep[k2] = 0.0f;  // E+ and E-
    __syncthreads();
    // ---- phase 1: this warp's two documents
    for (int s2 = 0; s2 < 2; s2++) {
      const int D = asg[2 * w + s2];
      const int k = D >> 5, dl = D & 31;  // (selects, not indexing: the arrays stay in registers)
      const uint32_t lmk = k ? lm[1] : lm[0];
      if (!((lmk >> dl) & 1u)) continue;
      const uint32_t cnt = __shfl_sync(kFull, k ? c_l[1] : c_l[0], dl);
      const int64_t eb = (k ? tb[1] : tb[0]) + __shfl_sync(kFull, k ? st_l[1] : st_l[0], dl);
      const int64_t id = (2 * T + k) * 32 + dl;
      float* Srow = S + D * kHQ;
      HeadTail<LOWER> cur = head_load<H, LOWER>(A, eb, 0, cnt, lane);
      for (int kk = lane; kk < m; kk += 32) {
        colU[kk] = __ldg(A.U + id * m + kk);
        if (LOWER) colL[kk] = __ldg(A.L + id * m + kk);
      }
      __syncwarp();
      for (uint32_t p0 = 0; p0 < cnt; p0 += 32) {
        HeadTail<LOWER> nxt;
        if (p0 + 32 < cnt) nxt = head_load<H, LOWER>(A, eb, p0 + 32, cnt, lane);
        const uint32_t j = cur.j;
        const uint32_t qb = cur.a.x;
        uint32_t nr = (cur.a.y & 0x3fffffffu) - qb;
        const bool head = (cur.b.x & kHeadMark) != 0;
        float eu = 0.0f, el = 0.0f;
        if (nr > 0 || head) {
          const uint4 da = cur.a;
          auto cell = [&](int o) -> int {
            if (H == 0) return (int)__ldg(A.pi + (int64_t)j * h + o);
            const uint32_t wv = o < 2 ? da.z : da.w;
            return (int)((o & 1) ? (wv >> 16) : (wv & 0xffffu));
          };
          if (da.y & (1u << 30)) eu = decode_upper_by(colU, h, cell);
          if (LOWER && (da.y & (1u << 31))) el = decode_lower_by(colL, h, cell);
        }
        if (head) {
          const int hh = (int)(cur.b.x & 0xffffu);
          Ep[hh * kHDocs + D] = eu;
          if (LOWER) Em[hh * kHDocs + D] = el;
        }
        // tail: wide terms walked by the whole warp (distinct, query-sorted), narrow ones lane-serial
        uint32_t wide = __ballot_sync(kFull, nr > (uint32_t)kNarrowMax);
        while (wide) {
          const int src = __ffs(wide) - 1;
          wide &= wide - 1;
          const uint32_t b = __shfl_sync(kFull, qb, src), nn = __shfl_sync(kFull, nr, src);
          const float wu = __shfl_sync(kFull, eu, src), wl = __shfl_sync(kFull, el, src);
          for (uint32_t r = lane; r < nn; r += 128) {
            uint2 pr[4];
#pragma unroll
            for (int u = 0; u < 4; u++)
              pr[u] = r + 32 * u < nn ? __ldg(A.pairs + b + r + 32 * u) : make_uint2(0, 0);
#pragma unroll
            for (int u = 0; u < 4; u++) {
              if (r + 32 * u < nn) {
                const float vv = __uint_as_float(pr[u].y);
                Srow[pr[u].x] = __fadd_rn(Srow[pr[u].x], __fmul_rn(vv, vv > 0.0f ? wu : wl));
              }
            }
          }
          __syncwarp();
        }
        if (nr > (uint32_t)kNarrowMax) nr = 0;
        const uint32_t maxr = __reduce_max_sync(kFull, nr);
        for (uint32_t r = 0; r < maxr; r++) {
          bool pend = r < nr;
          uint2 pr = make_uint2(0, 0);
          if (pend) {
            if (r == 0) pr = make_uint2(cur.b.x & 0x3ffu, cur.b.y);
            else if (r == 1) pr = make_uint2((cur.b.x >> 10) & 0x3ffu, cur.b.z);
            else if (r == 2) pr = make_uint2((cur.b.x >> 20) & 0x3ffu, cur.b.w);
            else pr = __ldg(A.pairs + qb + r);
          }
          const float vv = __uint_as_float(pr.y);
          const float c = __fmul_rn(vv, vv > 0.0f ? eu : el);
          const uint32_t qq = pr.x;
          // lanes holding the same query in one round: one winner per round (tag write/read)
          while (__any_sync(kFull, pend)) {
            if (pend) tag[qq] = (uint8_t)lane;
            __syncwarp();
            const bool win = pend && tag[qq] == (uint8_t)lane;
            if (win) Srow[qq] = __fadd_rn(Srow[qq], c);
            pend = pend && !win;
            __syncwarp();
          }
        }
        cur = nxt;
      }
      __syncwarp();
    }
    __syncthreads();
    // ---- phase 2: dense head product + compare; thread (half, q) owns query q of 32 documents
    if (qok) {
      float acc[32];
#pragma unroll
      for (int d = 0; d < 32; d++) {
        acc[d] = S[(32 * half + d) * kHQ + q];
        S[(32 * half + d) * kHQ + q] = 0.0f;
      }
#pragma unroll
      for (int hh = 0; hh < kHMax; hh++) {
        if (hh < hc) {
          const float vv = v[hh];
          const float4* row =
              reinterpret_cast<const float4*>(((LOWER && vv < 0.0f) ? Em : Ep) + hh * kHDocs + 32 * half);
#pragma unroll
          for (int d4 = 0; d4 < 8; d4++) {
            const float4 e4 = row[d4];
            acc[4 * d4 + 0] = fmaf(vv, e4.x, acc[4 * d4 + 0]);
            acc[4 * d4 + 1] = fmaf(vv, e4.y, acc[4 * d4 + 1]);
            acc[4 * d4 + 2] = fmaf(vv, e4.z, acc[4 * d4 + 2]);
            acc[4 * d4 + 3] = fmaf(vv, e4.w, acc[4 * d4 + 3]);
          }
        }
      }
      const uint32_t lmh = half ? lm[1] : lm[0];
#pragma unroll
      for (int d = 0; d < 32; d++) {
        const float x = acc[d] == 0.0f ? 0.0f : acc[d];
        if (((lmh >> d) & 1u) && x >= th)
          emit_h(A.cand, A.cand_cnt, A.cand_cap, (uint32_t)q, x, (uint32_t)((2 * T + half) * 32 + d));
      }
    } else {
#pragma unroll
      for (int d = 0; d < 32; d++) S[(32 * half + d) * kHQ + q] = 0.0f;
    }
    __syncthreads();
  }
}

// theta_q <- the k'-th largest score of a sample pass (its select output), if it has k' of them
__global__ void k_theta_from_sel(const float* __restrict__ cand_scores, int kprime, int nqc, float* __restrict__ theta) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nqc) return;
  const float s = cand_scores[(int64_t)q * kprime + kprime - 1];
  if (s != -INFINITY && s > theta[q]) theta[q] = s;
}

__global__ void k_fill_f32(float* p, float v, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

int num_sms_h() {
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

int head_max() { return kHMax; }
int head_cand_cap() { return kHeadCandCap; }

bool head_path_supported(int m, bool lower) { return head_smem_bytes(m, lower) <= 225 * 1024; }

int head_qmax() { return kHQ; }

void launch_head_select(const uint32_t* qoff, const int32_t* df, int32_t n, int64_t live, int64_t nq, float tau,
                        const uint2* pairs, uint4* dir, float* Qh, uint32_t* head_cnt, unsigned long long* hcand,
                        uint32_t* nhcand, int hmax, int qrow, cudaStream_t s) {
  cudaMemsetAsync(nhcand, 0, sizeof(uint32_t), s);
  const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8));
  k_head_cand<<<blocks, 256, 0, s>>>(qoff, df, n, 1.0f / (float)std::max<int64_t>(live, 1),
                                     1.0f / (float)std::max<int64_t>(nq, 1), tau, hcand, nhcand);
  k_head_pick<<<1, 1024, 0, s>>>(hcand, nhcand, qoff, pairs, dir, Qh, head_cnt, std::min(hmax, kHMax), qrow);
}

void launch_head_score(const int64_t* toff, const uint32_t* post, int64_t ntiles_total, int64_t stride,
                       const uint8_t* live, const int32_t* nnz, const float* U, const float* L, const uint16_t* pi,
                       int32_t m, int32_t h, const uint4* dir, const uint2* pairs, int32_t nqc, const float* theta,
                       const float* Qh, const uint32_t* head_cnt, unsigned long long* cand, uint32_t* cand_cnt,
                       uint32_t cand_cap, cudaStream_t s) {
  const int64_t n64 = (ntiles_total + 1) / 2;
  HeadArgs A{toff, post, ntiles_total, (n64 + stride - 1) / stride, stride, live, nnz, U, L, pi, m, h, dir, pairs,
             nqc, theta, Qh, head_cnt, cand, cand_cnt, cand_cap};
  const bool lower = L != nullptr;
  const size_t smem = head_smem_bytes(m, lower);
  const int H = h <= 4 ? h : 0;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(num_sms_h(), A.nvisit));
  static bool attr[5][2] = {};
  auto go = [&](void (*kern)(HeadArgs), int hh, int lo) {
    if (!attr[hh][lo]) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024);
      attr[hh][lo] = true;
    }
    kern<<<grid, 1024, smem, s>>>(A);
  };
#define SINN_HEAD_CASE(HH, LO) \
  if (H == HH && lower == LO) return go(k_head_score<HH, LO>, HH, LO);
  SINN_HEAD_CASE(0, false) SINN_HEAD_CASE(1, false) SINN_HEAD_CASE(2, false) SINN_HEAD_CASE(3, false)
  SINN_HEAD_CASE(4, false) SINN_HEAD_CASE(0, true) SINN_HEAD_CASE(1, true) SINN_HEAD_CASE(2, true)
  SINN_HEAD_CASE(3, true) SINN_HEAD_CASE(4, true)
#undef SINN_HEAD_CASE
}

void launch_theta_from_sel(const float* cand_scores, int kprime, int nqc, float* theta, cudaStream_t s) {
  k_theta_from_sel<<<(unsigned)((nqc + 255) / 256), 256, 0, s>>>(cand_scores, kprime, nqc, theta);
}

void launch_fill_theta(float* theta, float v, int n, cudaStream_t s) {
  k_fill_f32<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(theta, v, n);
}

}  // namespace sinn
