// NEXT row N1, literal per-direction form: the three direction systems A_i^M p_i = r_i^M of
// sizes M_i are solved by three solve launches (each padded to R_i = 8 ceil(M_i / 8), right-hand side in column
// i); this kernel places p_i into column i of the concatenated layout [p_1; p_2; p_3] (block i, zeros elsewhere;
// blocks start at SL-aligned offsets so the contraction kernel can skip them per b-group),
// which the contraction kernel reads with the cross-block operators [K_ij^M], [C_ij^M] -- argument
// placement only, no arithmetic.  A frequency whose direction solve failed gets NaN in all three columns (so every
// output entry of that frequency is NaN, as for a failed shared-basis solve) and the info code of the first failing
// column of the concatenation (M_1 + .. + M_{i-1} + k_i + 1), or -1 for a non-finite omega.
#include "podp_common.cuh"

namespace podp {

struct PerdirMap {
  const double2 *P[3];  // direction solves' P (F x 3 x R_i complex; column i holds p_i)
  int R[3];             // their padded sizes
  int m[3];             // M_i
  int offp[3];          // block offsets in the padded concatenation (the contraction kernel's rows)
  int off[3];           // block offsets in the unpadded concatenation (the P debug output)
};

__device__ __forceinline__ int32_t perdir_info(const int32_t *info3, int64_t F, int64_t f, const PerdirMap &mp) {
  const int32_t i0 = info3[f], i1 = info3[F + f], i2 = info3[2 * F + f];
  if (i0 == -1 || i1 == -1 || i2 == -1) return -1;
  const int32_t c0 = i0 > 0 ? i0 : 0x7fffffff, c1 = i1 > 0 ? mp.off[1] + i1 : 0x7fffffff,
                c2 = i2 > 0 ? mp.off[2] + i2 : 0x7fffffff;
  const int32_t cm = min(c0, min(c1, c2));
  return cm == 0x7fffffff ? 0 : cm;
}

__global__ void perdir_scatter_kernel(PerdirMap mp, const int32_t *__restrict__ info3, int64_t F,
                                      double2 *__restrict__ Pe, int Re, int32_t *__restrict__ info,
                                      double *__restrict__ P_out, int re) {
  const double nanv = __longlong_as_double(0x7ff8000000000000ll);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // padded concatenation for the contraction kernel
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < F * 3 * Re; g += stride) {
    const int64_t f = g / (3 * Re);
    const int rem = (int)(g - f * 3 * Re);
    const int i = rem / Re, k = rem - i * Re;
    const bool failed = info3[f] != 0 || info3[F + f] != 0 || info3[2 * F + f] != 0;
    double2 v = make_double2(0.0, 0.0);
    if (failed) v = make_double2(nanv, nanv);
    else if (k >= mp.offp[i] && k < mp.offp[i] + mp.m[i]) v = mp.P[i][(f * 3 + i) * mp.R[i] + (k - mp.offp[i])];
    Pe[(f * 3 + i) * Re + k] = v;
    if (info && rem == 0) info[f] = perdir_info(info3, F, f, mp);
  }
  // unpadded concatenation (PODP_FLAG_OUT_P): column i = (0, p_i, 0)
  if (P_out)
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < F * 3 * re; g += stride) {
      const int64_t f = g / (3 * re);
      const int rem = (int)(g - f * 3 * re);
      const int i = rem / re, k = rem - i * re;
      const bool failed = info3[f] != 0 || info3[F + f] != 0 || info3[2 * F + f] != 0;
      double2 v = make_double2(0.0, 0.0);
      if (failed) v = make_double2(nanv, nanv);
      else if (k >= mp.off[i] && k < mp.off[i] + mp.m[i]) v = mp.P[i][(f * 3 + i) * mp.R[i] + (k - mp.off[i])];
      P_out[g * 2] = v.x;
      P_out[g * 2 + 1] = v.y;
    }
}

cudaError_t launch_perdir_scatter(const double2 *const Pd[3], const int Rs[3], const int m[3], const int offp[3],
                                  const int32_t *info3, int64_t F, double2 *Pe, int Re, int32_t *info, double *P_out,
                                  cudaStream_t s) {
  PerdirMap mp;
  int re = 0;
  for (int i = 0; i < 3; ++i) {
    mp.P[i] = Pd[i];
    mp.R[i] = Rs[i];
    mp.m[i] = m[i];
    mp.offp[i] = offp[i];
    mp.off[i] = re;
    re += m[i];
  }
  const int64_t n = F * 3 * Re;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  perdir_scatter_kernel<<<(unsigned)blocks, 256, 0, s>>>(mp, info3, F, Pe, Re, info, P_out, re);
  return cudaGetLastError();
}

}  // namespace podp
