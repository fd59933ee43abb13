// sinn_device.cuh — device helpers shared by the scoring path and the debug decode kernel, so the
// decode the tests check bit-exactly is the one the scoring kernels run.
#pragma once
#include <stdint.h>

namespace sinn {

// A sketch cell as fp32: fp32 cells as stored; bfloat16 cells (F3, R21) are the upper 16 bits of
// the fp32 value (exact widening)
__device__ __forceinline__ float cellf(float v) { return v; }
__device__ __forceinline__ float cellf(uint16_t b) { return __uint_as_float((uint32_t)b << 16); }

// Least upper bound of x_i[j] (q_j > 0): min over the h upper cells pi_o(j) of column i (P:478-482,
// Alg. 6 line 8).  `col` points at U[i*m]; cell(o) returns pi_o(j), o < h.
template <class T, class Cell>
__device__ __forceinline__ float decode_upper_by(const T* __restrict__ col, int h, Cell cell) {
  float e = cellf(col[cell(0)]);
  for (int o = 1; o < h; o++) e = fminf(e, cellf(col[cell(o)]));
  return e;
}

// Greatest lower bound (q_j < 0): max over the h lower cells (Alg. 6 line 10).
template <class T, class Cell>
__device__ __forceinline__ float decode_lower_by(const T* __restrict__ col, int h, Cell cell) {
  float e = cellf(col[cell(0)]);
  for (int o = 1; o < h; o++) e = fmaxf(e, cellf(col[cell(o)]));
  return e;
}

template <class T>
__device__ __forceinline__ float decode_upper(const T* __restrict__ col, const int* cells, int h) {
  return decode_upper_by(col, h, [&](int o) { return cells[o]; });
}
template <class T>
__device__ __forceinline__ float decode_lower(const T* __restrict__ col, const int* cells, int h) {
  return decode_lower_by(col, h, [&](int o) { return cells[o]; });
}

// bfloat16 with directed rounding (R21): the smallest bfloat16 >= x (up) / largest <= x (down), as
// bits.  Representable values (low 16 bits zero, incl. +-inf) are kept; otherwise truncation (toward
// zero) is the rounding on one side and one bfloat16 step away from zero the rounding on the other.
__device__ __forceinline__ uint16_t bf16_up_bits(float x) {
  const uint32_t u = __float_as_uint(x);
  if ((u & 0xffffu) == 0) return (uint16_t)(u >> 16);
  const uint32_t t = (u >> 16) + ((u >> 31) ? 0u : 1u);
  return (uint16_t)t;
}
__device__ __forceinline__ uint16_t bf16_down_bits(float x) {
  const uint32_t u = __float_as_uint(x);
  if ((u & 0xffffu) == 0) return (uint16_t)(u >> 16);
  const uint32_t t = (u >> 16) + ((u >> 31) ? 1u : 0u);
  return (uint16_t)t;
}

// Order-preserving uint32 image of a float: larger float <=> larger key (-0 < +0; -inf lowest finite).
__device__ __forceinline__ uint32_t f2key(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float key2f(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

}  // namespace sinn

namespace sinn {

// ---- Tensor memory (TMEM, sm_100a tcgen05): 128 lanes x 512 columns x 32 bit per SM, read at
// ~700 B/clk/SM and written at ~640 B/clk/SM on the B200 (tools/mb/tmem.cu), off the L1/shared-memory
// pipe.  A warp reaches only the 32 lanes of its sub-partition (warp id % 4).  Used by k_doc_score to
// hold the batch's head-term query rows Q[hh][q] (read by every document's dense head product).
__device__ __forceinline__ void tmem_alloc512(uint32_t* smem_dst) {  // one whole warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
      (uint32_t)__cvta_generic_to_shared(smem_dst)));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
}
__device__ __forceinline__ void tmem_dealloc512(uint32_t taddr) {  // the allocating warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(taddr));
}
__device__ __forceinline__ void tmem_alloc32(uint32_t* smem_dst) {  // one whole warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;\n" ::"r"(
      (uint32_t)__cvta_generic_to_shared(smem_dst)));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
}
__device__ __forceinline__ void tmem_dealloc32(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;\n" ::"r"(taddr));
}
__device__ __forceinline__ void tmem_ld4(uint32_t taddr, float (&v)[4]) {
  uint32_t r[4];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 4; i++) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
// 16 consecutive columns of this thread's lane (32x32b shape: thread t <-> lane base + t)
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 16; i++) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 8; i++) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(
          taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15]))
      : "memory");
}

}  // namespace sinn
