// Latency of the LU pivot-column critical chain pieces on one warp, alone on the GPU (dev probe).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I ../paper_2307_05590_b200/csrc chain_probe.cu -o chain_probe
#include <cstdio>
#include "podp_common.cuh"
using namespace podp;

__device__ __forceinline__ double rcp_f32seed(double d) {
  // fp32 reciprocal seed (MUFU.RCP, ~23 bits) refined by two Newton steps in fp64
  double r = (double)__frcp_rn((float)d);
  double e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  return fma(r, e, r);
}

template <int KIND>
__global__ void probe(double2 *out, long long *cyc, int n) {
  double2 z = out[threadIdx.x];
  double2 u = make_double2(0.3, -0.2);
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (KIND == 0) {  // crecip_fast (MUFU.RCP64H + 2 Newton)
      z = crecip_fast(z);
    } else if (KIND == 1) {  // fp32-seeded reciprocal
      const double inv = rcp_f32seed(fma(z.x, z.x, z.y * z.y));
      z = make_double2(z.x * inv, -z.y * inv);
    } else if (KIND == 2) {  // cmul + cfms (the multiplier and the column update)
      z = cfms(cmul(z, u), u, z);
    } else if (KIND == 3) {  // double shuffle broadcast
      z.x = __shfl_sync(0xffffffffu, z.x, i & 31);
      z.y = __shfl_sync(0xffffffffu, z.y, (i + 1) & 31);
    } else if (KIND == 4) {  // redux.sync on an integer key derived from z
      unsigned k = (unsigned)(__double_as_longlong(z.x) >> 32);
      k = __reduce_max_sync(0xffffffffu, k);
      z.x = __hiloint2double((int)k, 0) ;
    } else if (KIND == 5) {  // full column chain: shfl p, recip, cmul, cfms, key, redux
      double2 p = make_double2(__shfl_sync(0xffffffffu, z.x, 3), __shfl_sync(0xffffffffu, z.y, 3));
      const double2 rc = crecip_fast(p);
      const double2 l = cmul(z, rc);
      z = cfms(l, u, z);
      unsigned k = (unsigned)(__double_as_longlong(z.x) >> 32) & 0x7fffffffu;
      k = __reduce_max_sync(0xffffffffu, k | (unsigned)threadIdx.x);
      z.y += (double)(k & 1);
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = z;
  if (threadIdx.x == 0) cyc[KIND] = t1 - t0;
}

int main() {
  double2 *d;
  long long *c, h[8];
  cudaMalloc(&d, 32 * sizeof(double2));
  cudaMalloc(&c, 8 * sizeof(long long));
  double2 init[32];
  for (int i = 0; i < 32; ++i) init[i] = make_double2(1.0 + 0.01 * i, 0.5);
  cudaMemcpy(d, init, sizeof(init), cudaMemcpyHostToDevice);
  const int n = 1000;
  for (int rep = 0; rep < 2; ++rep) {
    probe<0><<<1, 32>>>(d, c, n);
    probe<1><<<1, 32>>>(d, c, n);
    probe<2><<<1, 32>>>(d, c, n);
    probe<3><<<1, 32>>>(d, c, n);
    probe<4><<<1, 32>>>(d, c, n);
    probe<5><<<1, 32>>>(d, c, n);
    cudaDeviceSynchronize();
  }
  cudaMemcpy(h, c, 6 * sizeof(long long), cudaMemcpyDeviceToHost);
  const char *names[] = {"crecip_fast (MUFU.RCP64H + 2 Newton)", "fp32-seeded reciprocal", "cmul + cfms",
                         "double shuffle", "int key + redux.sync", "column chain (shfl, recip, cmul, cfms, redux)"};
  for (int k = 0; k < 6; ++k) printf("%-50s %6.1f clk per iteration\n", names[k], (double)h[k] / n);
  return 0;
}
