// Device helpers shared by the libpodp kernels (complex FP64 arithmetic on double2 = (re, im)).
// Every complex multiply-add is 4 DFMA (no Gauss 3M trick; SURVEY 7 "Parity is tight").
#pragma once
#include <cuda_runtime.h>
#include "podp_internal.h"

namespace podp {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// c + a*b
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 c) {
  return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}
// c - a*b
__device__ __forceinline__ double2 cfms(double2 a, double2 b, double2 c) {
  return make_double2(fma(-a.x, b.x, fma(a.y, b.y, c.x)), fma(-a.x, b.y, fma(-a.y, b.x, c.y)));
}
// c + conj(a)*b
__device__ __forceinline__ double2 cfma_conj(double2 a, double2 b, double2 c) {
  return make_double2(fma(a.x, b.x, fma(a.y, b.y, c.x)), fma(a.x, b.y, fma(-a.y, b.x, c.y)));
}
// 1/z = conj(z)/|z|^2 (IEEE division; no approximate reciprocal)
__device__ __forceinline__ double2 crecip(double2 z) {
  double d = fma(z.x, z.x, z.y * z.y);
  double inv = 1.0 / d;
  return make_double2(z.x * inv, -z.y * inv);
}
__device__ __forceinline__ double cabs1(double2 z) { return fabs(z.x) + fabs(z.y); }

// Entry order of the 6 unique entries (11,22,33,12,13,23) -- SPEC S:355.
__device__ __constant__ const int kPairI[6] = {0, 1, 2, 0, 0, 1};
__device__ __constant__ const int kPairJ[6] = {0, 1, 2, 1, 2, 2};

}  // namespace podp
