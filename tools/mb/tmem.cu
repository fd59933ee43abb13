// tools/mb/tmem.cu — TMEM read/write throughput on the B200 (tcgen05.ld / tcgen05.st, 32x32b.x32),
// against shared-memory LDS.128 reads of the same volume.  Question it answers: can a per-document
// dense head product read its query values Q[hh][q] from TMEM instead of shared memory (off the
// L1/shared-memory pipe that bounds k_doc_score on configs 3/5)?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb/tmem tools/mb/tmem.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int ITERS = 2048;

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
      "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
      "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
}

// MODE 0: tcgen05.ld (wait after each), 1: two loads in flight per wait, 2: tcgen05.st, 3: LDS.128
template <int MODE>
__global__ void __launch_bounds__(1024, 1) k_tmem(float* out, int iters) {
  __shared__ uint32_t taddr_s;
  __shared__ float4 sm[1024 * 2];  // 32 KB
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 1024 * 2; i += blockDim.x) sm[i] = make_float4(i, i + 1, i + 2, i + 3);
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&taddr_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tbase = taddr_s + ((uint32_t)(32 * (w & 3)) << 16);
  uint32_t acc = 0;
  float facc = 0.f;
  uint32_t v[32], u[32];
#pragma unroll
  for (int i = 0; i < 32; i++) v[i] = i + lane;
  for (int it = 0; it < iters; it++) {
    const uint32_t col = (uint32_t)((it * 32 + (w >> 2) * 64) & 511);
    if (MODE == 0) {
      tmem_ld32(tbase + col, v);
      asm volatile("tcgen05.wait::ld.sync.aligned;\n");
      acc ^= v[0] + v[31];
    } else if (MODE == 1) {
      tmem_ld32(tbase + col, v);
      tmem_ld32(tbase + ((col + 256) & 511), u);
      asm volatile("tcgen05.wait::ld.sync.aligned;\n");
      acc ^= v[0] + u[31];
      it++;
    } else if (MODE == 2) {
      v[0] = it;
      tmem_st32(tbase + col, v);
    } else {
      // 32 columns x 4 B per thread = 128 B per thread = eight LDS.128 (the same bytes as one x32 load)
#pragma unroll
      for (int k = 0; k < 8; k++) {
        const float4 a = sm[((it * 8 + k) * 32 + lane + w * 7) & (1024 * 2 - 1)];
        facc += a.x + a.w;
      }
    }
  }
  if (MODE == 2) asm volatile("tcgen05.wait::st.sync.aligned;\n");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(taddr_s));
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)acc + facc;
}

template <int MODE>
int run(const char* name, int sms, float* out) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  k_tmem<MODE><<<sms, 1024>>>(out, 16);
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(a));
  k_tmem<MODE><<<sms, 1024>>>(out, ITERS);
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, a, b));
  const double bytes = (double)sms * 32 * ITERS * 32 * 32 * 4;  // warps x iters x lanes x cols x 4 B
  int clk = 0;
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  const double cyc = ms * 1e-3 * clk * 1e3;
  printf("%-22s %8.3f ms  %8.1f GB/s chip  %7.1f B/clk/SM (at %d MHz)\n", name, ms, bytes / ms * 1e-6,
         bytes / sms / cyc, clk / 1000);
  return 0;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaFuncSetAttribute(k_tmem<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 0));
  float* out;
  CK(cudaMalloc(&out, sizeof(float) * sms * 1024));
  if (run<0>("tcgen05.ld x32", sms, out)) return 1;
  if (run<1>("tcgen05.ld x32 (2/wait)", sms, out)) return 1;
  if (run<2>("tcgen05.st x32", sms, out)) return 1;
  if (run<3>("LDS.128 same bytes", sms, out)) return 1;
  return 0;
}
