// sinn_device.cuh — device helpers shared by the scoring path and the debug decode kernel, so the
// decode the tests check bit-exactly is the one the scoring kernels run.
#pragma once
#include <stdint.h>

namespace sinn {

// Least upper bound of x_i[j] (q_j > 0): min over the h upper cells pi_o(j) of column i (P:478-482,
// Alg. 6 line 8).  `col` points at U[i*m]; cell(o) returns pi_o(j), o < h.
template <class Cell>
__device__ __forceinline__ float decode_upper_by(const float* __restrict__ col, int h, Cell cell) {
  float e = col[cell(0)];
  for (int o = 1; o < h; o++) e = fminf(e, col[cell(o)]);
  return e;
}

// Greatest lower bound (q_j < 0): max over the h lower cells (Alg. 6 line 10).
template <class Cell>
__device__ __forceinline__ float decode_lower_by(const float* __restrict__ col, int h, Cell cell) {
  float e = col[cell(0)];
  for (int o = 1; o < h; o++) e = fmaxf(e, col[cell(o)]);
  return e;
}

__device__ __forceinline__ float decode_upper(const float* __restrict__ col, const int* cells, int h) {
  return decode_upper_by(col, h, [&](int o) { return cells[o]; });
}
__device__ __forceinline__ float decode_lower(const float* __restrict__ col, const int* cells, int h) {
  return decode_lower_by(col, h, [&](int o) { return cells[o]; });
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
