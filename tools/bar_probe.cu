// Hand-off latency probe (dev tool): NW warps, step k produced by warp k % NW (bar.arrive), consumed by the
// others (bar.sync), as in the register-resident LU.  Variants: (0) bare hand-off, (1) + SHFL/recip/STS chain.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double rcp_nr(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  return fma(r, e, r);
}

template <int NW, int MODE>
__global__ void handoff(long long *out, double *sink) {
  __shared__ double buf[2][64];
  __shared__ int piv[2];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double x = 1.0 + lane, acc = 0;
  if (w == 0) { if (lane == 0) piv[0] = 0; buf[0][lane] = x; __syncwarp();
    asm volatile("bar.arrive %0, %1;" ::"r"(1), "r"(NW * 32) : "memory"); }
  long long t0 = clock64();
  for (int k = 0; k < 256; ++k) {
    const int wk = k % NW;
    if (w != wk) asm volatile("bar.sync %0, %1;" ::"r"(1 + (k & 1)), "r"(NW * 32) : "memory");
    const int p = piv[k & 1];
    double l = buf[k & 1][lane];
    acc += l * p;
    if (w == (k + 1) % NW) {
      double v = x + acc;
      if (MODE == 1) {
        v = __shfl_sync(0xffffffffu, v, (lane + 3) & 31);
        v = rcp_nr(v * v + 1.0) * v;
      }
      buf[(k + 1) & 1][lane] = v;
      if (lane == 0) piv[(k + 1) & 1] = k + 1;
      __syncwarp();
      asm volatile("bar.arrive %0, %1;" ::"r"(1 + ((k + 1) & 1)), "r"(NW * 32) : "memory");
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / 256;
  if (acc == 12345.0) sink[0] = acc;
}

int main() {
  long long *out; double *sink;
  cudaMallocManaged(&out, 8); cudaMalloc(&sink, 16);
  handoff<4, 0><<<1, 128>>>(out, sink); cudaDeviceSynchronize();
  printf("{\"probe\":\"handoff_nw4_bare\",\"clk_per_step\":%lld}\n", out[0]);
  handoff<4, 1><<<1, 128>>>(out, sink); cudaDeviceSynchronize();
  printf("{\"probe\":\"handoff_nw4_shfl_rcp\",\"clk_per_step\":%lld}\n", out[0]);
  handoff<2, 0><<<1, 64>>>(out, sink); cudaDeviceSynchronize();
  printf("{\"probe\":\"handoff_nw2_bare\",\"clk_per_step\":%lld}\n", out[0]);
  return 0;
}
