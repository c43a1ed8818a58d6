// N3 pencil solver kernel (PODP_FLAG_PENCIL): P(omega) = Z diag(1/(1 + i s lambda)) (c0 + omega c1), s = omega nu.
// Exact reformulation of eqn:ReducedA given the pencil precompute of pencil_host.cu; O(r^2) per
// frequency, no sequential dependency.  Z^T is staged in shared memory (conflict-free column reads); a block handles
// NF = floor(256 / R) frequencies at a time, thread (f, i) produces row i of P for frequency f (3 columns).
#include "podp_common.cuh"

namespace podp {

__global__ void __launch_bounds__(256) pencil_kernel(EvalArgs a) {
  extern __shared__ double2 smem[];
  const int R = a.L.R;
  const int NF = 256 / R;
  double2 *sZt = smem;                      // [R][R]: sZt[k*R + i] = Z[i][k]
  double2 *sY = sZt + (size_t)R * R;        // [NF][3][R]
  double *sLam = reinterpret_cast<double *>(sY + (size_t)NF * 3 * R);  // [R]
  const int64_t total = (int64_t)a.n_obj * a.F;
  const int tid = threadIdx.x;
  const int fl = tid / R, i = tid - fl * R;
  const bool active = fl < NF;
  const double nanv = __longlong_as_double(0x7ff8000000000000ll);
  int loaded = -1;
  const int64_t nchunks = (total + NF - 1) / NF;
  for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const int64_t t0 = ch * NF;
    const int obj0 = (int)(t0 / a.F);
    const int64_t tl = (t0 + NF - 1 < total ? t0 + NF - 1 : total - 1);
    const int obj1 = (int)(tl / a.F);
    // (re)load Z^T and lambda when the object changes (a chunk may straddle two objects: objects loaded per f)
    for (int ob = obj0; ob <= obj1; ++ob) {
      if (ob != loaded) {
        __syncthreads();
        const double *op = a.ops + (size_t)ob * a.L.stride;
        const double2 *gZ = reinterpret_cast<const double2 *>(op + a.L.Z);
        for (int e = tid; e < R * R; e += blockDim.x) {
          const int r = e / R, k = e - r * R;
          sZt[k * R + r] = gZ[e];
        }
        for (int e = tid; e < R; e += blockDim.x) sLam[e] = op[a.L.lam + e];
        __syncthreads();
        loaded = ob;
      }
      const int64_t t = t0 + fl;
      const bool mine = active && t < total && (int)(t / a.F) == ob;
      double2 *yv = sY + (size_t)(active ? fl : 0) * 3 * R;
      double w = 0.0;
      if (mine) {
        const int64_t f = t - (int64_t)ob * a.F;
        const double *op = a.ops + (size_t)ob * a.L.stride;
        w = a.omega[f];
        const double s = w * op[a.L.scal + SC_NU];
        const double2 *c0 = reinterpret_cast<const double2 *>(op + a.L.c0);
        const double2 *c1 = reinterpret_cast<const double2 *>(op + a.L.c1);
        // d = 1 / (1 + i s lambda_i)
        const double sl = s * sLam[i];
        const double den = 1.0 / fma(sl, sl, 1.0);
        const double2 d = make_double2(den, -sl * den);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double2 x0 = c0[c * R + i], x1 = c1[c * R + i];
          yv[c * R + i] = cmul(d, make_double2(fma(w, x1.x, x0.x), fma(w, x1.y, x0.y)));
        }
      }
      __syncthreads();
      if (mine) {
        double2 p0 = make_double2(0.0, 0.0), p1 = p0, p2 = p0;
        for (int k = 0; k < R; ++k) {
          const double2 z = sZt[k * R + i];
          p0 = cfma(z, yv[k], p0);
          p1 = cfma(z, yv[R + k], p1);
          p2 = cfma(z, yv[2 * R + k], p2);
        }
        const bool ok = isfinite(w);
        double2 *Pw = a.Pws + (size_t)t * 3 * R;
        Pw[i] = ok ? p0 : make_double2(nanv, nanv);
        Pw[R + i] = ok ? p1 : make_double2(nanv, nanv);
        Pw[2 * R + i] = ok ? p2 : make_double2(nanv, nanv);
        if (a.P_out && i < a.r) {
          double2 *Po = reinterpret_cast<double2 *>(a.P_out) + (size_t)t * 3 * a.r;
          Po[i] = Pw[i];
          Po[a.r + i] = Pw[R + i];
          Po[2 * a.r + i] = Pw[2 * R + i];
        }
        if (a.info && i == 0) a.info[t] = ok ? 0 : -1;
      }
      __syncthreads();
    }
  }
}

cudaError_t launch_pencil(const EvalArgs &a, cudaStream_t s) {
  const int R = a.L.R;
  if (R > 128) return cudaErrorNotSupported;
  const int NF = 256 / R;
  const size_t bytes = sizeof(double2) * ((size_t)R * R + (size_t)NF * 3 * R) + sizeof(double) * R;
  cudaError_t e = cudaFuncSetAttribute(pencil_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t total = (int64_t)a.n_obj * a.F;
  int64_t blocks = (total + NF - 1) / NF;
  const int per_sm = bytes > 110 * 1024 ? 1 : (bytes > 72 * 1024 ? 2 : 4);
  if (blocks > (int64_t)sms * per_sm) blocks = (int64_t)sms * per_sm;
  pencil_kernel<<<(unsigned)blocks, 256, bytes, s>>>(a);
  return cudaGetLastError();
}

}  // namespace podp

namespace podp {

// N3 fast path: y(omega) = diag(1/(1 + i s lambda)) (c0 + omega c1), s = omega nu -- O(r) per frequency; the
// MPT/certificate kernel then runs on y with the operators in pencil coordinates (podp_api.cu pencil_transform).
__global__ void __launch_bounds__(256) pencil_y_kernel(EvalArgs a) {
  const int R = a.L.R;
  const int64_t total = (int64_t)a.n_obj * a.F;
  const int64_t n = total * R;
  const double nanv = __longlong_as_double(0x7ff8000000000000ll);
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = g / R;
    const int b = (int)(g - t * R);
    const int obj = (int)(t / a.F);
    const int64_t f = t - (int64_t)obj * a.F;
    const double *op = a.ops + (size_t)obj * a.L.stride;
    const double w = a.omega[f];
    const bool ok = isfinite(w);
    const double sl = w * op[a.L.scal + SC_NU] * op[a.L.lam + b];
    const double den = 1.0 / fma(sl, sl, 1.0);
    const double2 d = make_double2(den, -sl * den);
    const double2 *c0 = reinterpret_cast<const double2 *>(op + a.L.c0);
    const double2 *c1 = reinterpret_cast<const double2 *>(op + a.L.c1);
    double2 *Pw = a.Pws + (size_t)t * 3 * R;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double2 x0 = c0[c * R + b], x1 = c1[c * R + b];
      const double2 y = cmul(d, make_double2(fma(w, x1.x, x0.x), fma(w, x1.y, x0.y)));
      Pw[c * R + b] = ok ? y : make_double2(nanv, nanv);
    }
    if (a.info && b == 0) a.info[t] = ok ? 0 : -1;
  }
}

cudaError_t launch_pencil_y(const EvalArgs &a, cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t n = (int64_t)a.n_obj * a.F * a.L.R;
  int64_t blocks = (n + 255) / 256;
  if (blocks > (int64_t)sms * 8) blocks = (int64_t)sms * 8;
  pencil_y_kernel<<<(unsigned)blocks, 256, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace podp
