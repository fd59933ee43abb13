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
