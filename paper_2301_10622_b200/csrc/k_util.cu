// k_util.cu — generic device primitives used by insert/delete: exclusive scans, a stable LSD
// radix sort of 64-bit keys (8-bit digits), fills.  Hand-written; no CUB/Thrust.
#include <algorithm>
#include <mutex>
#include <set>
#include <utility>

#include "sinn_internal.cuh"

namespace sinn {

int sm_count() {
  static int cache[256] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 256) dev = 0;
  if (!cache[dev]) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = n > 0 ? n : 1;
  }
  return cache[dev];
}

void smem_optin(const void* func) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (done.insert({func, dev}).second) {
    // the per-block maximum less the kernel's static shared memory (dynamic + static <= 227 KB)
    cudaFuncAttributes fa;
    int maxb = 0;
    cudaDeviceGetAttribute(&maxb, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (cudaFuncGetAttributes(&fa, func) == cudaSuccess && maxb > (int)fa.sharedSizeBytes)
      cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, maxb - (int)fa.sharedSizeBytes);
    cudaGetLastError();  // (a refused attribute surfaces as the launch's own error, not a stale one)
  }
}

namespace {

constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;                                // per thread
constexpr int kScanTile = kScanThreads * kScanItems;         // 4096

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t t = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= d) v += t;
  }
  return v;
}

// block-wide exclusive scan of one value per thread (NT <= 1024); *total = block sum
template <int NT>
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* total) {
  __shared__ uint32_t ws[NT / 32];
  __shared__ uint32_t tot;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t inc = warp_incl_scan(v);
  if (lane == 31) ws[w] = inc;
  __syncthreads();
  if (w == 0) {
    uint32_t x = lane < NT / 32 ? ws[lane] : 0;
    uint32_t xi = warp_incl_scan(x);
    if (lane < NT / 32) ws[lane] = xi - x;
    if (lane == 31) tot = xi;
  }
  __syncthreads();
  uint32_t ex = ws[w] + inc - v;
  *total = tot;
  __syncthreads();
  return ex;
}

__global__ void k_scan_reduce(const uint32_t* __restrict__ in, int64_t n, uint32_t* __restrict__ sums) {
  const int64_t base = (int64_t)blockIdx.x * kScanTile;
  uint32_t acc = 0;
#pragma unroll
  for (int t = 0; t < kScanItems; t++) {
    int64_t i = base + (int64_t)t * kScanThreads + threadIdx.x;
    if (i < n) acc += in[i];
  }
  uint32_t total;
  block_excl_scan<kScanThreads>(acc, &total);
  if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

// single block: exclusive scan of sums[0..nb) in place
__global__ void k_scan_sums(uint32_t* sums, int64_t nb) {
  uint32_t carry = 0;
  for (int64_t b0 = 0; b0 < nb; b0 += kScanThreads) {
    int64_t i = b0 + threadIdx.x;
    uint32_t v = i < nb ? sums[i] : 0;
    uint32_t total;
    uint32_t ex = block_excl_scan<kScanThreads>(v, &total);
    if (i < nb) sums[i] = carry + ex;
    carry += total;
  }
}

__global__ void k_scan_apply(const uint32_t* __restrict__ in, int64_t n, const uint32_t* __restrict__ sums,
                             uint32_t* __restrict__ out) {
  // each thread owns kScanItems consecutive elements (blocked arrangement) for an in-order scan
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  uint32_t v[kScanItems];
  uint32_t acc = 0;
#pragma unroll
  for (int t = 0; t < kScanItems; t++) {
    int64_t i = base + t;
    v[t] = i < n ? in[i] : 0;
    acc += v[t];
  }
  uint32_t total;
  uint32_t ex = block_excl_scan<kScanThreads>(acc, &total) + sums[blockIdx.x];
#pragma unroll
  for (int t = 0; t < kScanItems; t++) {
    int64_t i = base + t;
    if (i < n) out[i] = ex;
    ex += v[t];
  }
}

// single block exclusive scan of int64 (small n)
__global__ void k_scan_i64_small(const int64_t* __restrict__ in, int64_t* __restrict__ out, int64_t n) {
  __shared__ long long warp_sums[32];
  __shared__ long long carry_s;
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t b0 = 0; b0 < n; b0 += blockDim.x) {
    int64_t i = b0 + threadIdx.x;
    long long v = i < n ? in[i] : 0;
    long long inc = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      long long t = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= d) inc += t;
    }
    if (lane == 31) warp_sums[w] = inc;
    __syncthreads();
    if (w == 0) {
      long long x = lane < (int)(blockDim.x >> 5) ? warp_sums[lane] : 0;
      long long xi = x;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        long long t = __shfl_up_sync(0xffffffffu, xi, d);
        if (lane >= d) xi += t;
      }
      if (lane < (int)(blockDim.x >> 5)) warp_sums[lane] = xi - x;
    }
    __syncthreads();
    long long ex = carry_s + warp_sums[w] + inc - v;
    if (i < n) out[i] = ex;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry_s = ex + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) out[n] = carry_s;  // out has n+1 entries: out[n] = total
}

// one-CTA exclusive scan of a short u32 array (n outputs; in == out allowed): one launch instead of
// the three of the multi-block scan (the query-prep scan of small vocabularies)
__global__ void k_scan_u32_small(const uint32_t* in, uint32_t* out, int64_t n) {
  __shared__ uint32_t warp_sums[32];
  __shared__ uint32_t carry_s;
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t b0 = 0; b0 < n; b0 += blockDim.x) {
    int64_t i = b0 + threadIdx.x;
    uint32_t v = i < n ? in[i] : 0;
    uint32_t inc = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      uint32_t t = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= d) inc += t;
    }
    if (lane == 31) warp_sums[w] = inc;
    __syncthreads();
    if (w == 0) {
      uint32_t x = lane < (int)(blockDim.x >> 5) ? warp_sums[lane] : 0;
      uint32_t xi = x;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        uint32_t t = __shfl_up_sync(0xffffffffu, xi, d);
        if (lane >= d) xi += t;
      }
      if (lane < (int)(blockDim.x >> 5)) warp_sums[lane] = xi - x;
    }
    __syncthreads();
    uint32_t ex = carry_s + warp_sums[w] + inc - v;
    if (i < n) out[i] = ex;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry_s = ex + v;
    __syncthreads();
  }
}

// ---------------------------------------------------------------- radix sort (stable LSD, 8-bit digits)
constexpr int kRadixThreads = 256;
constexpr int kRadixWarps = kRadixThreads / 32;
constexpr int kRadixItemsPerWarp = 512;                     // 16 rounds of 32
constexpr int kRadixTile = kRadixWarps * kRadixItemsPerWarp;  // 4096

__global__ void k_radix_hist(const uint64_t* __restrict__ keys, int64_t n, int shift, uint32_t* __restrict__ hist,
                             int64_t nblocks) {
  __shared__ uint32_t h[256];
  for (int d = threadIdx.x; d < 256; d += blockDim.x) h[d] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kRadixTile;
  for (int t = threadIdx.x; t < kRadixTile; t += blockDim.x) {
    int64_t i = base + t;
    if (i < n) atomicAdd(&h[(uint32_t)(keys[i] >> shift) & 255u], 1u);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < 256; d += blockDim.x) hist[(int64_t)d * nblocks + blockIdx.x] = h[d];
}

__global__ void k_radix_scatter(const uint64_t* __restrict__ keys, int64_t n, int shift,
                                const uint32_t* __restrict__ offs, int64_t nblocks, uint64_t* __restrict__ out) {
  __shared__ uint32_t wcount[kRadixWarps][256];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int d = lane; d < 256; d += 32) wcount[w][d] = 0;
  __syncwarp();
  const int64_t wbase = (int64_t)blockIdx.x * kRadixTile + (int64_t)w * kRadixItemsPerWarp;
  constexpr int kRounds = kRadixItemsPerWarp / 32;
  uint64_t key[kRounds];
  uint32_t pos[kRounds];  // position within the warp's items of the same digit
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int r = 0; r < kRounds; r++) {
    int64_t i = wbase + r * 32 + lane;
    bool valid = i < n;
    key[r] = valid ? keys[i] : 0;
    uint32_t d = valid ? (uint32_t)(key[r] >> shift) & 255u : 256u + 0u;
    uint32_t peers = __match_any_sync(0xffffffffu, d);
    uint32_t rank = __popc(peers & lt);
    uint32_t before = valid ? wcount[w][d] : 0;
    __syncwarp();
    if (valid && rank == 0) wcount[w][d] = before + __popc(peers);
    __syncwarp();
    pos[r] = before + rank;
  }
  __syncthreads();
  // exclusive prefix over warps per digit, plus this block's global base
  __shared__ uint32_t wpre[kRadixWarps][256];
  for (int d = threadIdx.x; d < 256; d += blockDim.x) {
    uint32_t acc = offs[(int64_t)d * nblocks + blockIdx.x];
#pragma unroll
    for (int ww = 0; ww < kRadixWarps; ww++) {
      wpre[ww][d] = acc;
      acc += wcount[ww][d];
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kRounds; r++) {
    int64_t i = wbase + r * 32 + lane;
    if (i < n) {
      uint32_t d = (uint32_t)(key[r] >> shift) & 255u;
      out[wpre[w][d] + pos[r]] = key[r];
    }
  }
}

__global__ void k_fill_u8(uint8_t* p, uint8_t v, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}
__global__ void k_fill_f32(float* p, float v, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}
__global__ void k_fill_u16(uint16_t* p, uint16_t v, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

inline unsigned grid_for(int64_t n, int threads, int cap_blocks = 0) {
  if (cap_blocks <= 0) cap_blocks = sm_count() * 16;
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > cap_blocks) b = cap_blocks;
  return (unsigned)b;
}

}  // namespace

size_t exclusive_scan_u32_tmp_elems(int64_t n) { return (size_t)((n + kScanTile - 1) / kScanTile) + 1; }

void exclusive_scan_u32(const uint32_t* in, uint32_t* out, int64_t n, uint32_t* tmp, cudaStream_t s) {
  if (n <= 0) return;
  if (n <= 4096) {
    k_scan_u32_small<<<1, 1024, 0, s>>>(in, out, n);
    return;
  }
  int64_t nb = (n + kScanTile - 1) / kScanTile;
  k_scan_reduce<<<(unsigned)nb, kScanThreads, 0, s>>>(in, n, tmp);
  k_scan_sums<<<1, kScanThreads, 0, s>>>(tmp, nb);
  k_scan_apply<<<(unsigned)nb, kScanThreads, 0, s>>>(in, n, tmp, out);
}

// multi-block exclusive scan of int64 (out has n + 1 entries: out[n] = total): per-block sums of 4,096
// elements, one block scans the sums, each block applies its carry.  (Round 1 used one 1,024-thread
// block for the whole array: 0.13 ms per call over config 5's 125 K tiles, three calls per insert.)
constexpr int kScan64Tile = 4096;
__global__ void __launch_bounds__(1024) k_scan64_reduce(const int64_t* __restrict__ in, int64_t n,
                                                        long long* __restrict__ sums) {
  __shared__ long long ws[32];
  const int64_t b0 = (int64_t)blockIdx.x * kScan64Tile;
  long long v = 0;
  for (int k = 0; k < kScan64Tile / 1024; k++) {
    const int64_t i = b0 + k * 1024 + threadIdx.x;
    if (i < n) v += in[i];
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    long long x = ws[threadIdx.x];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) x += __shfl_xor_sync(0xffffffffu, x, d);
    if (threadIdx.x == 0) sums[blockIdx.x] = x;
  }
}

__global__ void __launch_bounds__(1024) k_scan64_apply(const int64_t* __restrict__ in, int64_t n,
                                                       const long long* __restrict__ carry, int64_t* __restrict__ out) {
  __shared__ long long ws[32];
  __shared__ long long base;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t b0 = (int64_t)blockIdx.x * kScan64Tile;
  if (threadIdx.x == 0) base = carry[blockIdx.x];
  __syncthreads();
  // thread t owns elements [b0 + 4t, b0 + 4t + 4)
  long long v[4], loc = 0;
#pragma unroll
  for (int k = 0; k < 4; k++) {
    const int64_t i = b0 + 4 * threadIdx.x + k;
    v[k] = i < n ? in[i] : 0;
    loc += v[k];
  }
  long long inc = loc;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const long long y = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += y;
  }
  if (lane == 31) ws[w] = inc;
  __syncthreads();
  if (w == 0) {
    const long long x = ws[lane];
    long long xi = x;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, xi, d);
      if (lane >= d) xi += y;
    }
    ws[lane] = xi - x;
  }
  __syncthreads();
  long long run = base + ws[w] + inc - loc;
#pragma unroll
  for (int k = 0; k < 4; k++) {
    const int64_t i = b0 + 4 * threadIdx.x + k;
    if (i < n) out[i] = run;
    run += v[k];
  }
  if (b0 + kScan64Tile >= n && threadIdx.x == 1023) out[n] = run;  // the last block writes the total
}

void exclusive_scan_i64_small(const int64_t* in, int64_t* out, int64_t n, cudaStream_t s) {
  const int64_t nb = (n + kScan64Tile - 1) / kScan64Tile;
  if (nb <= 1) {
    k_scan_i64_small<<<1, 1024, 0, s>>>(in, out, n);
    return;
  }
  // block sums: a grow-only stream-ordered scratch per device
  static long long* scratch[256] = {};
  static int64_t have[256] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 256) dev = 0;
  if (have[dev] < nb + 1) {
    if (scratch[dev]) cudaFreeAsync(scratch[dev], s);
    have[dev] = std::max<int64_t>(nb + 1, 1 << 14);
    cudaMallocAsync((void**)&scratch[dev], sizeof(long long) * (size_t)have[dev], s);
  }
  long long* sums = scratch[dev];
  k_scan64_reduce<<<(unsigned)nb, 1024, 0, s>>>(in, n, sums);
  k_scan_i64_small<<<1, 1024, 0, s>>>(reinterpret_cast<const int64_t*>(sums), reinterpret_cast<int64_t*>(sums), nb);
  k_scan64_apply<<<(unsigned)nb, 1024, 0, s>>>(in, n, sums, out);
}

size_t radix_sort_hist_elems(int64_t n) { return (size_t)256 * (size_t)((n + kRadixTile - 1) / kRadixTile); }

// Sorts keys[0..n) by bits [lo_bit, hi_bit) (stable); result ends in `keys` (tmp is scratch of n).
void radix_sort_u64(uint64_t* keys, uint64_t* tmp, int64_t n, int lo_bit, int hi_bit, uint32_t* hist,
                    uint32_t* scan_tmp, cudaStream_t s) {
  if (n <= 1 || hi_bit <= lo_bit) return;
  int64_t nb = (n + kRadixTile - 1) / kRadixTile;
  uint64_t* src = keys;
  uint64_t* dst = tmp;
  int passes = 0;
  for (int shift = lo_bit; shift < hi_bit; shift += 8, passes++) {
    k_radix_hist<<<(unsigned)nb, kRadixThreads, 0, s>>>(src, n, shift, hist, nb);
    exclusive_scan_u32(hist, hist, 256 * nb, scan_tmp, s);
    k_radix_scatter<<<(unsigned)nb, kRadixThreads, 0, s>>>(src, n, shift, hist, nb, dst);
    uint64_t* t = src; src = dst; dst = t;
  }
  if (passes & 1) cudaMemcpyAsync(keys, src, sizeof(uint64_t) * (size_t)n, cudaMemcpyDeviceToDevice, s);
}

void fill_u8(uint8_t* p, uint8_t v, int64_t n, cudaStream_t s) {
  if (n > 0) k_fill_u8<<<grid_for(n, 256), 256, 0, s>>>(p, v, n);
}
// out += sum of v[i] over i < n, with w[i] != 0 when w is given (int64 accumulation)
__global__ void k_sum_i32(const int32_t* __restrict__ v, const uint8_t* __restrict__ w, int64_t n,
                          unsigned long long* __restrict__ out) {
  long long acc = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (!w || w[i]) acc += v[i];
  for (int d = 16; d > 0; d >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, d);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, (unsigned long long)acc);
}
void launch_sum_i32(const int32_t* v, const uint8_t* w, int64_t n, int64_t* out, cudaStream_t s) {
  cudaMemsetAsync(out, 0, sizeof(int64_t), s);
  if (n > 0) k_sum_i32<<<grid_for(n, 256), 256, 0, s>>>(v, w, n, reinterpret_cast<unsigned long long*>(out));
}

__global__ void k_fault_probe() {}
void launch_fault_probe(cudaStream_t s) { k_fault_probe<<<1, 1025, 0, s>>>(); }

void fill_f32(float* p, float v, int64_t n, cudaStream_t s) {
  if (n > 0) k_fill_f32<<<grid_for(n, 256), 256, 0, s>>>(p, v, n);
}
void fill_u16(uint16_t* p, uint16_t v, int64_t n, cudaStream_t s) {
  if (n > 0) k_fill_u16<<<grid_for(n, 256), 256, 0, s>>>(p, v, n);
}

}  // namespace sinn
