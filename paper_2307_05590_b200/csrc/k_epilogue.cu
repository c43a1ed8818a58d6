// NEXT row N4: per-frequency epilogues on the MPT outputs.
//   * tensor invariants: eigenvalues of Rt and of I (ascending), the rotation-invariant features used for
//     dictionary matching ("the eigenvalues of the real and imaginary parts of the MPT");
//   * coil-pair voltages V ~ (H0^ms)_i (Rt + i I)_ij (H0)_j for given background fields (eqn:meas_voltage,
//     P:393-395).
// One thread per output row; HBM-bound (48 B + 48 B in, 48 B or 16 n_coil B out per row).
#include "podp_common.cuh"

namespace podp {

// eigenvalues of a real symmetric 3x3 matrix (6 entries, order 11,22,33,12,13,23) by cyclic Jacobi, ascending
__device__ __forceinline__ void eig3_sym(const double *t6, double *ev) {
  double a[3][3] = {{t6[0], t6[3], t6[4]}, {t6[3], t6[1], t6[5]}, {t6[4], t6[5], t6[2]}};
#pragma unroll 1
  for (int sweep = 0; sweep < 12; ++sweep) {
    const double off = fabs(a[0][1]) + fabs(a[0][2]) + fabs(a[1][2]);
    const double scale = fabs(a[0][0]) + fabs(a[1][1]) + fabs(a[2][2]) + off;
    if (off == 0.0 || off <= 1e-18 * scale) break;
#pragma unroll
    for (int pq = 0; pq < 3; ++pq) {
      const int p = pq == 2 ? 1 : 0, q = pq == 0 ? 1 : 2;
      const double apq = a[p][q];
      if (apq == 0.0) continue;
      const double theta = 0.5 * atan2(2.0 * apq, a[q][q] - a[p][p]);
      const double c = cos(theta), s = sin(theta);
      // A <- J^T A J with J = [[c, s], [-s, c]] on (p, q): zeroes a[p][q]
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double akp = a[k][p], akq = a[k][q];
        a[k][p] = c * akp - s * akq;
        a[k][q] = s * akp + c * akq;
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double apk = a[p][k], aqk = a[q][k];
        a[p][k] = c * apk - s * aqk;
        a[q][k] = s * apk + c * aqk;
      }
      a[p][q] = a[q][p] = 0.0;
    }
  }
  double e0 = a[0][0], e1 = a[1][1], e2 = a[2][2], tmp;
  if (e0 > e1) { tmp = e0; e0 = e1; e1 = tmp; }
  if (e1 > e2) { tmp = e1; e1 = e2; e2 = tmp; }
  if (e0 > e1) { tmp = e0; e0 = e1; e1 = tmp; }
  ev[0] = e0;
  ev[1] = e1;
  ev[2] = e2;
}

__global__ void invariants_kernel(const double *__restrict__ T1, const double *__restrict__ I, int64_t n,
                                  double *__restrict__ eigR, double *__restrict__ eigI) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    double r6[6], i6[6], ev[3];
#pragma unroll
    for (int e = 0; e < 6; ++e) {
      r6[e] = T1[t * 6 + e];
      i6[e] = I[t * 6 + e];
    }
    eig3_sym(r6, ev);
#pragma unroll
    for (int e = 0; e < 3; ++e) eigR[t * 3 + e] = ev[e];
    eig3_sym(i6, ev);
#pragma unroll
    for (int e = 0; e < 3; ++e) eigI[t * 3 + e] = ev[e];
  }
}

__global__ void coil_voltage_kernel(const double *__restrict__ T1, const double *__restrict__ I, int64_t n,
                                    const double *__restrict__ hex, const double *__restrict__ hms, int n_coil,
                                    double2 *__restrict__ V) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    double m[3][3][2];
    const int ii[6] = {0, 1, 2, 0, 0, 1}, jj[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
    for (int e = 0; e < 6; ++e) {
      const double re = T1[t * 6 + e], im = I[t * 6 + e];
      m[ii[e]][jj[e]][0] = m[jj[e]][ii[e]][0] = re;
      m[ii[e]][jj[e]][1] = m[jj[e]][ii[e]][1] = im;
    }
    for (int c = 0; c < n_coil; ++c) {
      double vr = 0.0, vi = 0.0;
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          const double w = hms[c * 3 + i] * hex[c * 3 + j];
          vr = fma(w, m[i][j][0], vr);
          vi = fma(w, m[i][j][1], vi);
        }
      V[t * n_coil + c] = make_double2(vr, vi);
    }
  }
}

cudaError_t launch_invariants(const double *T1, const double *I, int64_t n, double *eigR, double *eigI, cudaStream_t s) {
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  invariants_kernel<<<(unsigned)blocks, 256, 0, s>>>(T1, I, n, eigR, eigI);
  return cudaGetLastError();
}

cudaError_t launch_coil_voltage(const double *T1, const double *I, int64_t n, const double *hex_d, const double *hms_d,
                                int n_coil, double *V, cudaStream_t s) {
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  coil_voltage_kernel<<<(unsigned)blocks, 256, 0, s>>>(T1, I, n, hex_d, hms_d, n_coil, reinterpret_cast<double2 *>(V));
  return cudaGetLastError();
}

}  // namespace podp
