// tools/mb/mb.cu — micro-benchmarks that calibrate the round-2 scoring-kernel design on the B200:
// FFMA / FFMA2 issue rates, the dense-head inner loop (LDS.128 broadcast + FFMA), shared-memory
// read-modify-write (LDS + FADD + STS, conflict-free), and SHFL throughput.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb/mb tools/mb/mb.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int ITERS = 4096;

__global__ void k_ffma(float* out, float a, float b) {
  float acc[16];
#pragma unroll
  for (int i = 0; i < 16; i++) acc[i] = threadIdx.x * 0.001f + i;
  float q = a + threadIdx.x;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 16; i++) acc[i] = fmaf(q, acc[(i + 1) & 15], acc[i]);  // 3 regs
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; i++) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// GEMM-like: acc[d] += q * e[d] with 32 accumulators, e[] 8 regs reused
__global__ void k_ffma_gemm(float* out, float a) {
  float acc[32], e[8];
#pragma unroll
  for (int i = 0; i < 32; i++) acc[i] = 0.f;
#pragma unroll
  for (int i = 0; i < 8; i++) e[i] = threadIdx.x * 0.01f + i;
  float q0 = a, q1 = a * 0.5f, q2 = a * 0.25f, q3 = a * 0.125f;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int d = 0; d < 8; d++) {
      acc[d] = fmaf(q0, e[d], acc[d]);
      acc[8 + d] = fmaf(q1, e[d], acc[8 + d]);
      acc[16 + d] = fmaf(q2, e[d], acc[16 + d]);
      acc[24 + d] = fmaf(q3, e[d], acc[24 + d]);
    }
    q0 += 1e-7f;
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 32; i++) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ffma2(float* out, float a) {
  float2 acc[16];
#pragma unroll
  for (int i = 0; i < 16; i++) acc[i] = make_float2(threadIdx.x * 0.001f + i, i);
  float2 q = make_float2(a, a * 0.5f);
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 16; i++) acc[i] = __ffma2_rn(q, acc[(i + 1) & 15], acc[i]);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; i++) s += acc[i].x + acc[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// dense-head inner loop: thread = 1 query x 32 docs; per head term hh: q from smem (per lane),
// E row of 32 docs (LDS.128 x 8, warp-broadcast), 32 FFMA
__global__ void __launch_bounds__(1024, 1) k_dense(float* out, int H) {
  extern __shared__ float sm[];
  float* E = sm;             // [H][32]
  float* Q = sm + H * 32;    // [H][1024]
  for (int i = threadIdx.x; i < H * 32; i += blockDim.x) E[i] = i * 1e-3f;
  for (int i = threadIdx.x; i < H * 1024; i += blockDim.x) Q[i] = i * 1e-4f;
  __syncthreads();
  float acc[32];
#pragma unroll
  for (int i = 0; i < 32; i++) acc[i] = 0.f;
  for (int it = 0; it < ITERS / 16; it++) {
    for (int hh = 0; hh < H; hh++) {
      const float q = Q[hh * 1024 + threadIdx.x];
      const float4* e4 = reinterpret_cast<const float4*>(E + hh * 32);
#pragma unroll
      for (int k = 0; k < 8; k++) {
        float4 e = e4[k];
        acc[4 * k] = fmaf(q, e.x, acc[4 * k]);
        acc[4 * k + 1] = fmaf(q, e.y, acc[4 * k + 1]);
        acc[4 * k + 2] = fmaf(q, e.z, acc[4 * k + 2]);
        acc[4 * k + 3] = fmaf(q, e.w, acc[4 * k + 3]);
      }
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 32; i++) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// dense variant: thread = 2 queries x 16 docs (E 4x LDS.128 broadcast, Q LDS.64)
__global__ void __launch_bounds__(1024, 1) k_dense2(float* out, int H) {
  extern __shared__ float sm[];
  float* E = sm;             // [H][32]
  float* Q = sm + H * 32;    // [H][1024]
  for (int i = threadIdx.x; i < H * 32; i += blockDim.x) E[i] = i * 1e-3f;
  for (int i = threadIdx.x; i < H * 1024; i += blockDim.x) Q[i] = i * 1e-4f;
  __syncthreads();
  float acc[32];
#pragma unroll
  for (int i = 0; i < 32; i++) acc[i] = 0.f;
  const int qp = threadIdx.x & 511, half = threadIdx.x >> 9;
  for (int it = 0; it < ITERS / 16; it++) {
    for (int hh = 0; hh < H; hh++) {
      const float2 q = reinterpret_cast<const float2*>(Q + hh * 1024)[qp];
      const float4* e4 = reinterpret_cast<const float4*>(E + hh * 32 + 16 * half);
#pragma unroll
      for (int k = 0; k < 4; k++) {
        float4 e = e4[k];
        acc[4 * k] = fmaf(q.x, e.x, acc[4 * k]);
        acc[4 * k + 1] = fmaf(q.x, e.y, acc[4 * k + 1]);
        acc[4 * k + 2] = fmaf(q.x, e.z, acc[4 * k + 2]);
        acc[4 * k + 3] = fmaf(q.x, e.w, acc[4 * k + 3]);
        acc[16 + 4 * k] = fmaf(q.y, e.x, acc[16 + 4 * k]);
        acc[16 + 4 * k + 1] = fmaf(q.y, e.y, acc[16 + 4 * k + 1]);
        acc[16 + 4 * k + 2] = fmaf(q.y, e.z, acc[16 + 4 * k + 2]);
        acc[16 + 4 * k + 3] = fmaf(q.y, e.w, acc[16 + 4 * k + 3]);
      }
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 32; i++) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// shared-memory RMW: S[d][q] += v * e with lane = query (conflict-free), d rotating
__global__ void __launch_bounds__(1024, 1) k_rmw(float* out) {
  extern __shared__ float S[];  // [32][1024]
  for (int i = threadIdx.x; i < 32 * 1024; i += blockDim.x) S[i] = 0.f;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const float v = lane * 0.01f;
  int q = w * 32 + lane;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int d = 0; d < 8; d++) {
      float* p = S + ((d + it) & 31) * 1024 + q;
      *p = fmaf(v, 1.0001f, *p);
    }
  }
  __syncthreads();
  out[blockIdx.x * blockDim.x + threadIdx.x] = S[threadIdx.x];
}

__global__ void k_shfl(float* out) {
  float x = threadIdx.x, y = 0;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int k = 0; k < 8; k++) y += __shfl_sync(0xffffffffu, x, (k + it) & 31);
    x += 1e-7f;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = y;
}

int main() {
  float* out;
  CK(cudaMalloc(&out, 148 * 2 * 1024 * 4 * 4));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int dev = 0, clk = 0, sms = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  printf("SMs %d clock %d kHz\n", sms, clk);
  auto time = [&](const char* name, auto launch, double ops_per_thread, int threads, int blocks) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int r = 0; r < 5; r++) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ms /= 5;
    double ops = ops_per_thread * threads * (double)blocks;
    printf("%-28s %8.3f ms  %8.2f T ops/s  (%.1f ops/clk/SM at %.0f MHz nominal)  err=%s\n", name, ms, ops / ms / 1e9,
           ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1e3, cudaGetErrorString(cudaGetLastError()));
  };
  const int B = sms, T = 1024;
  time("FFMA 3-reg", [&] { k_ffma<<<B * 2, T>>>(out, 1.f, 2.f); }, 16.0 * ITERS, T, B * 2);
  time("FFMA gemm 4x8", [&] { k_ffma_gemm<<<B * 2, T / 2>>>(out, 1.f); }, 32.0 * ITERS, T / 2, B * 2);
  time("FFMA2 (x2 flops)", [&] { k_ffma2<<<B * 2, T>>>(out, 1.f); }, 32.0 * ITERS, T, B * 2);
  for (int H : {8, 16}) {
    size_t sm = (size_t)H * (32 + 1024) * 4;
    cudaFuncSetAttribute(k_dense, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaFuncSetAttribute(k_dense2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    char nm[64];
    snprintf(nm, 64, "dense 1qx32d H=%d (FMA)", H);
    time(nm, [&] { k_dense<<<B, T, sm>>>(out, H); }, 32.0 * H * (ITERS / 16), T, B);
    snprintf(nm, 64, "dense 2qx16d H=%d (FMA)", H);
    time(nm, [&] { k_dense2<<<B, T, sm>>>(out, H); }, 32.0 * H * (ITERS / 16), T, B);
  }
  cudaFuncSetAttribute(k_rmw, cudaFuncAttributeMaxDynamicSharedMemorySize, 32 * 1024 * 4);
  time("smem RMW (updates)", [&] { k_rmw<<<B, T, 32 * 1024 * 4>>>(out); }, 8.0 * ITERS, T, B);
  time("SHFL", [&] { k_shfl<<<B * 2, T>>>(out); }, 8.0 * ITERS, T, B * 2);
  return 0;
}
