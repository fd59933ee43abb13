// k_delete.cu — deletion: ids become vacant and every instance is removed from the
// inverted lists (order-preserving per-term compaction); the sketch column stays stale until
// the id is recycled.  Also the stand-alone decode kernel used for bit-exact decode parity.
#include "sinn_device.cuh"
#include <algorithm>

#include "sinn_internal.cuh"

namespace sinn {

namespace {

__global__ void k_mark_vacant(const uint32_t* __restrict__ ids, int64_t count, uint8_t* __restrict__ live) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < count; r += (int64_t)gridDim.x * blockDim.x)
    live[ids[r]] = 0;
}

// one block per tile: number of entries of tile t whose document is still live (order-agnostic)
__global__ void k_count_live(const int64_t* __restrict__ off, const uint32_t* __restrict__ post,
                             const uint8_t* __restrict__ live, int64_t n, int64_t* __restrict__ counts) {
  __shared__ int64_t part[32];
  for (int64_t j = blockIdx.x; j < n; j += gridDim.x) {
    const int64_t b = off[j], e = off[j + 1];
    int64_t c = 0;
    for (int64_t p = b + threadIdx.x; p < e; p += blockDim.x) c += live[(j << 5) | (post[p] & 31u)];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) c += __shfl_xor_sync(0xffffffffu, c, d);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
      int64_t t = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); w++) t += part[w];
      counts[j] = t;
    }
    __syncthreads();
  }
}

// one block per tile: stable compaction of the live entries of tile t to new_post[new_off[t] ..)
__global__ void k_compact(const int64_t* __restrict__ off, const uint32_t* __restrict__ post,
                          const uint8_t* __restrict__ live, int64_t n, const int64_t* __restrict__ new_off,
                          uint32_t* __restrict__ new_post, int32_t* __restrict__ df) {
  __shared__ uint32_t wsum[32];
  __shared__ int64_t carry;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int64_t j = blockIdx.x; j < n; j += gridDim.x) {
    const int64_t b = off[j], e = off[j + 1];
    uint32_t* out = new_post + new_off[j];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t t0 = b; t0 < e; t0 += blockDim.x) {
      const int64_t p = t0 + threadIdx.x;
      uint32_t id = 0;
      bool keep = false;
      if (p < e) {
        id = post[p];
        keep = live[(j << 5) | (id & 31u)] != 0;
        if (!keep) atomicSub(&df[id >> 5], 1);  // the entry of a deleted document leaves I[term]
      }
      const uint32_t bal = __ballot_sync(0xffffffffu, keep);
      const uint32_t rank = __popc(bal & ((1u << lane) - 1u));
      if (lane == 0) wsum[w] = __popc(bal);
      __syncthreads();
      uint32_t before = 0, total = 0;
      for (int ww = 0; ww < nw; ww++) {
        if (ww < w) before += wsum[ww];
        total += wsum[ww];
      }
      if (keep) out[carry + before + rank] = id;
      __syncthreads();
      if (threadIdx.x == 0) carry += total;
      __syncthreads();
    }
  }
}

template <class T>  // sketch cell: float, or bfloat16 bits (F3)
__global__ void k_decode(const uint32_t* __restrict__ ids, const int32_t* __restrict__ terms,
                         const uint8_t* __restrict__ positive, int64_t count, const T* __restrict__ U,
                         const T* __restrict__ L, const uint16_t* __restrict__ pi, int32_t m, int32_t h,
                         int upper_only, float* __restrict__ out) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x) {
    const int32_t j = terms[t];
    int cells[SINN_MAX_H];
    for (int o = 0; o < h; o++) cells[o] = pi[(int64_t)j * h + o];
    float e;
    if (positive[t]) e = decode_upper(U + (int64_t)ids[t] * m, cells, h);
    else if (upper_only) e = 0.0f;
    else e = decode_lower(L + (int64_t)ids[t] * m, cells, h);
    out[t] = e;
  }
}

template <class T>
__global__ void k_gather_rows(const uint32_t* __restrict__ ids, int64_t count, const T* __restrict__ src,
                              int32_t m, float* __restrict__ out) {
  const int64_t total = count * m;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x)
    out[t] = cellf(src[(int64_t)ids[t / m] * m + t % m]);
}

inline unsigned grid_for(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > (int64_t)sm_count() * 32) b = (int64_t)sm_count() * 32;
  return (unsigned)b;
}

}  // namespace

void launch_mark_vacant(const uint32_t* ids, int64_t count, uint8_t* live, cudaStream_t s) {
  k_mark_vacant<<<grid_for(count, 256), 256, 0, s>>>(ids, count, live);
}

void launch_count_live_postings(const int64_t* off, const uint32_t* post, const uint8_t* live, int64_t n,
                                int64_t* counts, cudaStream_t s) {
  int64_t blocks = std::min<int64_t>(n, (int64_t)sm_count() * 64);
  if (blocks < 1) blocks = 1;
  k_count_live<<<(unsigned)blocks, 256, 0, s>>>(off, post, live, n, counts);
}

void launch_compact_postings(const int64_t* off, const uint32_t* post, const uint8_t* live, int64_t n,
                             const int64_t* new_off, uint32_t* new_post, int32_t* df, cudaStream_t s) {
  int64_t blocks = std::min<int64_t>(n, (int64_t)sm_count() * 64);
  if (blocks < 1) blocks = 1;
  k_compact<<<(unsigned)blocks, 256, 0, s>>>(off, post, live, n, new_off, new_post, df);
}

// export of I[term] from the tile-major index: inside a tile the entries are grouped by document,
// so the (at most one per document) entries of `term` are found by a linear scan of the tile; they
// come out in ascending id order.
__global__ void k_term_count(const int64_t* __restrict__ off, const uint32_t* __restrict__ post, int64_t ntiles,
                             uint32_t term, uint32_t* __restrict__ cnt) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < ntiles; t += (int64_t)gridDim.x * blockDim.x) {
    uint32_t c = 0;
    for (int64_t p = off[t]; p < off[t + 1]; p++) c += (post[p] >> 5) == term;
    cnt[t] = c;
  }
}

__global__ void k_term_write(const int64_t* __restrict__ off, const uint32_t* __restrict__ post, int64_t ntiles,
                             uint32_t term, const uint32_t* __restrict__ pos, uint32_t* __restrict__ out,
                             int64_t cap) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < ntiles; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t w = pos[t];
    for (int64_t p = off[t]; p < off[t + 1]; p++) {
      const uint32_t e = post[p];
      if ((e >> 5) != term) continue;
      if (w < cap) out[w] = (uint32_t)((t << 5) | (e & 31u));
      w++;
    }
  }
}

void launch_export_term(const int64_t* off, const uint32_t* post, int64_t ntiles, uint32_t term, uint32_t* cnt,
                        uint32_t* pos, uint32_t* scan_tmp, uint32_t* out, int64_t cap, cudaStream_t s) {
  if (ntiles <= 0) return;
  k_term_count<<<grid_for(ntiles, 256), 256, 0, s>>>(off, post, ntiles, term, cnt);
  exclusive_scan_u32(cnt, pos, ntiles + 1, scan_tmp, s);
  k_term_write<<<grid_for(ntiles, 256), 256, 0, s>>>(off, post, ntiles, term, pos, out, cap);
}

void launch_gather_rows(const uint32_t* ids, int64_t count, const void* src, bool bf16, int32_t m, float* out,
                        cudaStream_t s) {
  if (count <= 0) return;
  if (bf16)
    k_gather_rows<<<grid_for(count * m, 256), 256, 0, s>>>(ids, count, (const uint16_t*)src, m, out);
  else
    k_gather_rows<<<grid_for(count * m, 256), 256, 0, s>>>(ids, count, (const float*)src, m, out);
}

void launch_decode(const uint32_t* ids, const int32_t* terms, const uint8_t* positive, int64_t count,
                   const void* U, const void* L, bool bf16, const uint16_t* pi, int32_t m, int32_t h,
                   bool upper_only, float* out, cudaStream_t s) {
  if (count <= 0) return;
  if (bf16)
    k_decode<<<grid_for(count, 256), 256, 0, s>>>(ids, terms, positive, count, (const uint16_t*)U,
                                                   (const uint16_t*)L, pi, m, h, upper_only ? 1 : 0, out);
  else
    k_decode<<<grid_for(count, 256), 256, 0, s>>>(ids, terms, positive, count, (const float*)U, (const float*)L,
                                                   pi, m, h, upper_only ? 1 : 0, out);
}

}  // namespace sinn
