// k_head.cu — head-term selection of a query batch (part of S0, Alg. 6 lines 1-2):
// the terms whose expected coverage of (document, query) pairs is largest become the per-document
// dense head product of k_doc_score (k_doc.cuh): their query values go to dense rows Qh[hh][q] and
// their directory sector is marked, so the walk records their decoded estimates instead of walking
// their long query lists.  Coverage of term j = df[j]/live x (queries of the pass holding j)/nq.
#include <stdint.h>

#include <algorithm>

#include "sinn_internal.cuh"

namespace sinn {

namespace {

constexpr int kHCand = 4096;   // head candidates considered per pass
constexpr int kHeadMax = 16;   // head terms per pass (the most k_doc_score's TMEM rows hold)

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
// the query lacks j), and the term's mark in k_doc_score's 32-byte directory sector (no sparse pairs,
// head mark | hh)
__global__ void __launch_bounds__(1024) k_head_pick(const unsigned long long* __restrict__ cand,
                                                    const uint32_t* __restrict__ ncand,
                                                    const uint32_t* __restrict__ qoff, const uint2* __restrict__ pairs,
                                                    uint4* __restrict__ dir,
                                                    float* __restrict__ Qh, uint32_t* __restrict__ head_cnt, int hmax,
                                                    int qrow) {
  __shared__ unsigned long long sb[kHCand];
  __shared__ uint32_t hj[kHeadMax];
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
  const int hc = (int)min(cnt, (uint32_t)min(hmax, kHeadMax));
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
  }
  if (threadIdx.x == 0) *head_cnt = (uint32_t)hc;
}


}  // namespace

int head_cand_cap() { return kHCand; }

void launch_head_select(const uint32_t* qoff, const int32_t* df, int32_t n, int64_t live, int64_t nq, float tau,
                        const uint2* pairs, uint4* dir, float* Qh, uint32_t* head_cnt, unsigned long long* hcand,
                        uint32_t* nhcand, int hmax, int qrow, cudaStream_t s) {
  cudaMemsetAsync(nhcand, 0, sizeof(uint32_t), s);
  const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)sm_count() * 8));
  k_head_cand<<<blocks, 256, 0, s>>>(qoff, df, n, 1.0f / (float)std::max<int64_t>(live, 1),
                                     1.0f / (float)std::max<int64_t>(nq, 1), tau, hcand, nhcand);
  k_head_pick<<<1, 1024, 0, s>>>(hcand, nhcand, qoff, pairs, dir, Qh, head_cnt, std::min(hmax, kHeadMax), qrow);
}

}  // namespace sinn
