// K2: batched shifted complex LU + 3-RHS solve, rows a2-a3 of SURVEY 8(a).
//   A(omega) = K + i omega nu M,  B(omega) = b0 + omega b1,  P = A^{-1} B        (eqn:ReducedA)
// Generic path: one warp per (object, omega); the augmented matrix [A | B] (R x (R+3) complex) lives in shared
// memory; right-looking LU with partial pivoting (max |re|+|im|, lowest index on ties, as LAPACK izamax),
// warp-shuffle argmax, rank-1 updates spread over the warp, then back substitution.  Writes P (3 x R per omega,
// direction-major) to the hand-off workspace consumed by K3.
#include "podp_common.cuh"

namespace podp {

// GLOBAL = true keeps [A | B] in a per-warp global-memory scratch (L1/L2 cached) instead of shared memory: the
// fallback for R too large for a warp's shared-memory slice (R > ~118).
template <int NW, bool GLOBAL>
__global__ void __launch_bounds__(NW * 32) solve_smem_kernel(EvalArgs a, double2 *gscratch) {
  extern __shared__ double2 smem[];
  const int R = a.L.R;
  const int LD = R + 4;  // R + 3 columns, +1 pad
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2 *A = GLOBAL ? gscratch + ((size_t)blockIdx.x * NW + warp) * R * LD : smem + (size_t)warp * R * LD;
  const int64_t total = (int64_t)a.n_obj * a.F;
  const bool pivot = !(a.flags & PODP_FLAG_NO_PIVOT);

  for (int64_t t = (int64_t)blockIdx.x * NW + warp; t < total; t += (int64_t)gridDim.x * NW) {
    const int obj = (int)(t / a.F);
    const int64_t f = t - (int64_t)obj * a.F;
    const double *op = a.ops + (size_t)obj * a.L.stride;
    const double w = a.omega[f];
    const double s = w * op[a.L.scal + SC_NU];
    const double2 *K = reinterpret_cast<const double2 *>(op + a.L.K);
    const double2 *M = reinterpret_cast<const double2 *>(op + a.L.M);
    const double2 *b0 = reinterpret_cast<const double2 *>(op + a.L.b0);
    const double2 *b1 = reinterpret_cast<const double2 *>(op + a.L.b1);
    // a2: assemble A = K + i s M and B = b0 + w b1
    for (int e = lane; e < R * R; e += 32) {
      const int i = e / R, j = e - i * R;
      const double2 k = K[e], m = M[e];
      A[i * LD + j] = make_double2(fma(-s, m.y, k.x), fma(s, m.x, k.y));
    }
    for (int e = lane; e < 3 * R; e += 32) {
      const int c = e / R, i = e - c * R;
      const double2 x0 = b0[e], x1 = b1[e];
      A[i * LD + R + c] = make_double2(fma(w, x1.x, x0.x), fma(w, x1.y, x0.y));
    }
    __syncwarp();
    int info = isfinite(w) ? 0 : -1;
    // a3: LU with partial pivoting on [A | B] (forward elimination of B rides along)
    for (int k = 0; k < R && info == 0; ++k) {
      int p = k;
      if (pivot) {
        double best = -1.0;
        for (int i = k + lane; i < R; i += 32) {
          const double m = cabs1(A[i * LD + k]);
          if (m > best) { best = m; p = i; }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          const double ob = __shfl_xor_sync(0xffffffffu, best, o);
          const int op_ = __shfl_xor_sync(0xffffffffu, p, o);
          if (ob > best || (ob == best && op_ < p)) { best = ob; p = op_; }
        }
        if (!(best > 0.0)) { info = k + 1; break; }  // exactly zero (or NaN) pivot column
        if (p != k) {
          for (int j = lane; j < R + 3; j += 32) {
            const double2 x = A[k * LD + j];
            A[k * LD + j] = A[p * LD + j];
            A[p * LD + j] = x;
          }
          __syncwarp();
        }
      } else {
        const double2 d = A[k * LD + k];
        if (d.x == 0.0 && d.y == 0.0) { info = k + 1; break; }
      }
      const double2 rc = crecip_scaled(A[k * LD + k]);  // range-safe (no |p|^2 under/overflow)
      for (int i = k + 1 + lane; i < R; i += 32) A[i * LD + k] = cmul(A[i * LD + k], rc);
      __syncwarp();
      const int nr = R - k - 1, nc = R + 3 - k - 1;
      for (int e = lane; e < nr * nc; e += 32) {
        const int ii = e / nc, jj = e - ii * nc;
        const int i = k + 1 + ii, j = k + 1 + jj;
        A[i * LD + j] = cfms(A[i * LD + k], A[k * LD + j], A[i * LD + j]);
      }
      __syncwarp();
    }
    // back substitution U x = y (3 right-hand sides in columns R..R+2)
    if (info == 0) {
      for (int k = R - 1; k >= 0; --k) {
        const double2 rc = crecip_scaled(A[k * LD + k]);  // range-safe (no |p|^2 under/overflow)
        __syncwarp();
        if (lane < 3) A[k * LD + R + lane] = cmul(A[k * LD + R + lane], rc);
        __syncwarp();
        for (int e = lane; e < 3 * k; e += 32) {
          const int i = e / 3, c = e - 3 * i;
          A[i * LD + R + c] = cfms(A[i * LD + k], A[k * LD + R + c], A[i * LD + R + c]);
        }
        __syncwarp();
      }
    }
    const double nan = __longlong_as_double(0x7ff8000000000000ll);
    double2 *Pw = a.Pws + (size_t)t * 3 * R;
    for (int e = lane; e < 3 * R; e += 32) {
      const int c = e / R, i = e - c * R;
      Pw[e] = info == 0 ? A[i * LD + R + c] : make_double2(nan, nan);
    }
    if (a.P_out) {
      double2 *Po = reinterpret_cast<double2 *>(a.P_out) + (size_t)t * 3 * a.r;
      for (int e = lane; e < 3 * a.r; e += 32) {
        const int c = e / a.r, i = e - c * a.r;
        Po[e] = info == 0 ? A[i * LD + R + c] : make_double2(nan, nan);
      }
    }
    if (a.info && lane == 0) a.info[t] = info;
    __syncwarp();
  }
}

size_t solve_scratch_bytes(int R, int sms) {
  const size_t per_warp = (size_t)R * (R + 4) * sizeof(double2);
  return per_warp > 200 * 1024 ? per_warp * (size_t)sms * 4 : 0;
}

cudaError_t launch_solve(const EvalArgs &a, cudaStream_t s, double2 *gscratch) {
  const int R = a.L.R;
  const size_t per_warp = (size_t)R * (R + 4) * sizeof(double2);
  int dev0 = 0, sms0 = 148;
  cudaGetDevice(&dev0);
  cudaDeviceGetAttribute(&sms0, cudaDevAttrMultiProcessorCount, dev0);
  if (per_warp > 200 * 1024) {  // global-memory scratch fallback: one warp per block, 4 blocks per SM
    if (!gscratch) return cudaErrorInvalidValue;
    const int64_t total = (int64_t)a.n_obj * a.F;
    int64_t blocks = total < (int64_t)sms0 * 4 ? total : (int64_t)sms0 * 4;
    solve_smem_kernel<1, true><<<(unsigned)blocks, 32, 0, s>>>(a, gscratch);
    return cudaGetLastError();
  }
  int nw = (int)((200 * 1024) / per_warp);
  if (nw > 8) nw = 8;
  if (nw < 1) nw = 1;
  const int64_t total = (int64_t)a.n_obj * a.F;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaError_t e;
#define PODP_LAUNCH_SOLVE(NWv)                                                                              \
  {                                                                                                         \
    const size_t sm = per_warp * NWv;                                                                       \
    e = cudaFuncSetAttribute(solve_smem_kernel<NWv, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
    if (e != cudaSuccess) return e;                                                                         \
    int64_t blocks = (total + NWv - 1) / NWv;                                                               \
    int64_t cap = (int64_t)sms * 8;                                                                         \
    if (blocks > cap) blocks = cap;                                                                         \
    solve_smem_kernel<NWv, false><<<(unsigned)blocks, NWv * 32, sm, s>>>(a, nullptr);                       \
  }
  if (nw >= 8) PODP_LAUNCH_SOLVE(8)
  else if (nw >= 4) PODP_LAUNCH_SOLVE(4)
  else if (nw >= 2) PODP_LAUNCH_SOLVE(2)
  else PODP_LAUNCH_SOLVE(1)
#undef PODP_LAUNCH_SOLVE
  return cudaGetLastError();
}

}  // namespace podp
