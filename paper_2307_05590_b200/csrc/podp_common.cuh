// Device helpers shared by the libpodp kernels (complex FP64 arithmetic on double2 = (re, im)).
// Every complex multiply-add here is 4 DFMA.  (Gauss's three-product form is used only in the DMMA trailing updates of
// the left-looking LU for 32 <= R <= 80, k_lu_ll.cu body<M3>; DESIGN reading B14 has the measured parity margins.)
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

// 1/d for a normal, finite d > 0: hardware reciprocal seed (MUFU.RCP64H, ~2^-23) refined by two Newton steps
// (relative error ~1 ulp).  Used on the LU pivot critical path instead of the IEEE division sequence (which adds
// a slow-path branch and ~2x the latency).  Out-of-range d (|p| < 1e-150 or > 1e150) yields inf/0 and the
// affected frequency is flagged non-finite downstream.
__device__ __forceinline__ double rcp_nr(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  return fma(r, e, r);
}
__device__ __forceinline__ double2 crecip_fast(double2 z) {
  const double inv = rcp_nr(fma(z.x, z.x, z.y * z.y));
  return make_double2(z.x * inv, -z.y * inv);
}
// 1/z for any finite nonzero z without a division or a call: z is scaled by the exact power of two 2^(1023-E)
// (E = biased exponent of max(|Re|,|Im|), clamped to 2045) into max(|Re|,|Im|) in [1, 2) (or a smaller normal
// value when z is subnormal), so |z'|^2 is a normal number for rcp_nr, and the scale is applied once more to the
// result: 1/z = conj(z') / |z'|^2 * 2^(1023-E).  Overflows to inf only when 1/|z| is not representable (as the
// IEEE quotient would).  Used where crecip_fast's |z|^2 leaves the normal range.
__device__ __forceinline__ double2 crecip_scaled(double2 z) {
  const unsigned hx = (unsigned)(__double_as_longlong(z.x) >> 32) & 0x7FF00000u;
  const unsigned hy = (unsigned)(__double_as_longlong(z.y) >> 32) & 0x7FF00000u;
  const unsigned h = min(hx > hy ? hx : hy, 0x7FD00000u);  // E << 20, E <= 2045
  const double sc = __hiloint2double((int)(0x7FE00000u - h), 0);  // 2^(1023 - E), exact
  const double zx = z.x * sc, zy = z.y * sc;
  const double inv = rcp_nr(fma(zx, zx, zy * zy));
  return make_double2(zx * inv * sc, -zy * inv * sc);
}

// Pivot magnitude key: max(|Re|, |Im|) from the high words of the doubles (sign cleared), i.e. exponent + top
// 20 mantissa bits, computed on the integer pipe.  Monotone in max(|Re|,|Im|) up to 2^-20 relative.
__device__ __forceinline__ unsigned mag_key_hi(double2 z) {
  const unsigned hr = (unsigned)(__double_as_longlong(z.x) >> 32) & 0x7FFFFFFFu;
  const unsigned hi = (unsigned)(__double_as_longlong(z.y) >> 32) & 0x7FFFFFFFu;
  return hr > hi ? hr : hi;
}

// Entry order of the 6 unique entries (11,22,33,12,13,23) -- SPEC S:355.
__device__ __constant__ const int kPairI[6] = {0, 1, 2, 0, 0, 1};
__device__ __constant__ const int kPairJ[6] = {0, 1, 2, 1, 2, 2};

}  // namespace podp
