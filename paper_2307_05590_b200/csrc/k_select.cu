// K4: greedy argmax-error reduction, row a7 of SURVEY 8(a): one step of Algorithm 1.
//   Lambda_n = max_{omega_n <= omega < omega_{n+1}, i<=j} Delta_ij(omega)   (last interval closed, reading U12)
//   Lambda = max_n Lambda_n; choose the N* largest (ties -> lower n), or Lambda_n >= theta*Lambda.
// Pass 1 reduces the per-interval maximum (exact FP64 compare via the order-preserving bit pattern of a
// non-negative double, warp-aggregated 64-bit atomicMax), pass 2 the lowest grid index attaining it
// (atomicMin), pass 3 (one warp) the top-N* choice.  HBM-bound: 48 B of Delta + 8 B of omega per grid point.
#include "podp_common.cuh"

namespace podp {

__device__ __forceinline__ int find_interval(const double *snap, int n_snap, double w) {
  // returns interval index n in [0, n_snap-2], or -1 if w is not a candidate
  if (!(w >= snap[0]) || !(w <= snap[n_snap - 1])) return -1;
  int lo = 0, hi = n_snap - 1;  // invariant snap[lo] <= w, answer = largest n with snap[n] <= w
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (snap[mid] <= w) lo = mid; else hi = mid;
  }
  if (snap[lo] == w) return -1;                       // equals a snapshot
  if (lo >= n_snap - 1) return -1;
  if (lo + 1 <= n_snap - 1 && snap[lo + 1] == w) return -1;
  return lo;
}

__device__ __forceinline__ unsigned long long point_key(const double *D6) {
  double v = -1.0;
#pragma unroll
  for (int e = 0; e < 6; ++e) {
    const double d = D6[e];
    if (d == d && d > v) v = d;  // NaN ignored
  }
  if (v < 0.0) return 0ull;      // no finite non-negative entry
  v = v + 0.0;                   // canonicalise -0.0
  return (unsigned long long)__double_as_longlong(v) + 1ull;  // 0 reserved for "empty"
}

__global__ void select_max_kernel(const double *__restrict__ omega, const double *__restrict__ Delta, int64_t F,
                                  const double *__restrict__ snap, int n_snap, unsigned long long *lam_key) {
  extern __shared__ double s_snap[];
  for (int i = threadIdx.x; i < n_snap; i += blockDim.x) s_snap[i] = snap[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < F; base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t f = base + threadIdx.x;
    int n = -1;
    unsigned long long key = 0;
    if (f < F) {
      n = find_interval(s_snap, n_snap, omega[f]);
      if (n >= 0) key = point_key(Delta + f * 6);
      if (key == 0) n = -1;
    }
    // warp-aggregated atomicMax per interval
    unsigned active = __ballot_sync(0xffffffffu, n >= 0);
    while (active) {
      const int leader = __ffs(active) - 1;
      const int nl = __shfl_sync(0xffffffffu, n, leader);
      unsigned long long v = (n == nl) ? key : 0ull;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const unsigned long long ov = __shfl_xor_sync(0xffffffffu, v, o);
        v = ov > v ? ov : v;
      }
      if (lane == leader) atomicMax(lam_key + nl, v);
      active &= ~__ballot_sync(0xffffffffu, n == nl);
    }
  }
}

__global__ void select_arg_kernel(const double *__restrict__ omega, const double *__restrict__ Delta, int64_t F,
                                  const double *__restrict__ snap, int n_snap, const unsigned long long *lam_key,
                                  unsigned long long *arg_idx) {
  extern __shared__ double s_snap[];
  for (int i = threadIdx.x; i < n_snap; i += blockDim.x) s_snap[i] = snap[i];
  __syncthreads();
  for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < F; f += (int64_t)gridDim.x * blockDim.x) {
    const int n = find_interval(s_snap, n_snap, omega[f]);
    if (n < 0) continue;
    const unsigned long long key = point_key(Delta + f * 6);
    if (key != 0ull && key == lam_key[n]) atomicMin(arg_idx + n, (unsigned long long)f);
  }
}

// result layout (doubles): [0] n_new, [1] Lambda, [2 .. 2+n_int) Lambda_n (-1 = empty),
// then n_star grid indices, then n_star omegas (both ascending by index; unused slots -1 / NaN).
__global__ void select_final_kernel(const double *__restrict__ omega, int n_int, int n_star, double theta,
                                    const unsigned long long *g_lam_key, const unsigned long long *g_arg_idx,
                                    double *result) {
  // the per-interval keys and indices are staged in shared memory by the whole block first (independent loads), so
  // the serial choice below does not wait on one L2 round trip per read
  extern __shared__ unsigned long long s_ka[];
  unsigned long long *lam_key = s_ka, *arg_idx = s_ka + n_int;
  for (int n = threadIdx.x; n < n_int; n += blockDim.x) {
    lam_key[n] = g_lam_key[n];
    arg_idx[n] = g_arg_idx[n];
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  double lam_g = -1.0;
  int n_cand = 0;
  for (int n = 0; n < n_int; ++n) {
    const unsigned long long k = lam_key[n];
    const double v = k ? __longlong_as_double((long long)(k - 1ull)) : -1.0;
    result[2 + n] = v;
    if (k) { ++n_cand; if (v > lam_g) lam_g = v; }
  }
  result[1] = lam_g;
  double *idx = result + 2 + n_int, *om = idx + n_star;
  for (int q = 0; q < n_star; ++q) { idx[q] = -1.0; om[q] = __longlong_as_double(0x7ff8000000000000ll); }
  if (n_cand == 0 || (theta <= 0.0 && n_cand < n_star)) { result[0] = -1.0; return; }
  // pick up to n_star intervals by (-Lambda_n, n), optionally thresholded (n_star <= 64 enforced by the host)
  long long chosen[64];
  int chosen_n[64];
  int nc = 0;
  for (int q = 0; q < n_star; ++q) {
    int best = -1;
    double bv = -1.0;
    for (int n = 0; n < n_int; ++n) {
      const unsigned long long k = lam_key[n];
      if (!k) continue;
      bool taken = false;
      for (int t = 0; t < nc; ++t) taken |= (chosen_n[t] == n);
      if (taken) continue;
      const double v = __longlong_as_double((long long)(k - 1ull));
      if (theta > 0.0 && !(v >= theta * lam_g)) continue;
      if (v > bv) { bv = v; best = n; }   // strict > keeps the lower n on ties
    }
    if (best < 0) break;
    chosen_n[nc] = best;
    chosen[nc++] = (long long)arg_idx[best];
  }
  // sort chosen grid indices ascending
  for (int a = 1; a < nc; ++a) {
    long long x = chosen[a];
    int b = a - 1;
    while (b >= 0 && chosen[b] > x) { chosen[b + 1] = chosen[b]; --b; }
    chosen[b + 1] = x;
  }
  for (int q = 0; q < nc; ++q) { idx[q] = (double)chosen[q]; om[q] = omega[chosen[q]]; }
  result[0] = (double)nc;
}

cudaError_t launch_select(const double *omega, const double *Delta, int64_t F, const double *snap_d, int n_snap,
                          int n_star, double theta, unsigned long long *lam_key, unsigned long long *arg_idx,
                          double *result_d, cudaStream_t s, int *nlaunch) {
  const int n_int = n_snap - 1;
  cudaError_t e = cudaMemsetAsync(lam_key, 0, sizeof(unsigned long long) * n_int, s);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(arg_idx, 0xff, sizeof(unsigned long long) * n_int, s);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t blocks = (F + 255) / 256;
  if (blocks > (int64_t)sms * 8) blocks = (int64_t)sms * 8;
  if (blocks < 1) blocks = 1;
  const size_t sm = sizeof(double) * n_snap;
  select_max_kernel<<<(unsigned)blocks, 256, sm, s>>>(omega, Delta, F, snap_d, n_snap, lam_key);
  select_arg_kernel<<<(unsigned)blocks, 256, sm, s>>>(omega, Delta, F, snap_d, n_snap, lam_key, arg_idx);
  select_final_kernel<<<1, 128, 2 * sizeof(unsigned long long) * n_int, s>>>(omega, n_int, n_star, theta, lam_key,
                                                                             arg_idx, result_d);
  *nlaunch += 3;
  return cudaGetLastError();
}

}  // namespace podp
