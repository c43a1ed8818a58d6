// Latency probes (dev tool): dependent-chain latency of the ops on the LU pivot critical path, alone and with
// 3 other warps per SMSP streaming DFMAs.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double2 crecip(double2 z) {
  double d = fma(z.x, z.x, z.y * z.y);
  double inv = 1.0 / d;
  return make_double2(z.x * inv, -z.y * inv);
}

template <int OP>
__global__ void probe(long long *out, double *sink, int load_warps) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp >= 4) {  // background DFMA load (warps 4..): same SMSPs as warps 0..3
    if (warp - 4 >= load_warps * 4) return;
    double acc[8];
    for (int c = 0; c < 8; ++c) acc[c] = lane * 1e-9 + c;
    for (int i = 0; i < 4000; ++i)
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[c] = fma(acc[c], 0.999999, 1e-7);
    double s = 0; for (int c = 0; c < 8; ++c) s += acc[c];
    if (s == 1.0) sink[0] = s;
    return;
  }
  if (warp != 0) return;
  double x = 1.0 + lane * 1e-3;
  double2 z = make_double2(3.0 + lane, 1.0);
  unsigned key = lane;
  float f = 1.0f;
  __syncwarp();
  long long t0 = clock64();
  for (int it = 0; it < 256; ++it) {
    if (OP == 0) x = fma(x, 0.9999, 1e-7);                                     // DFMA chain
    if (OP == 1) { z = crecip(z); }                                             // complex reciprocal
    if (OP == 2) { key = __reduce_max_sync(0xffffffffu, key) + lane; }          // CREDUX
    if (OP == 3) { x = __shfl_sync(0xffffffffu, x, (lane + 1) & 31); }          // SHFL double (2x32)
    if (OP == 4) { f = __double2float_rn(x + f); x = (double)f; }               // F2F pair
    if (OP == 5) { x = 1.0 / x; }                                               // IEEE double reciprocal
  }
  long long t1 = clock64();
  if (lane == 0) out[0] = (t1 - t0) / 256;
  if (x == 12345.0 || z.x == 3.0 || key == 7 || f == 2.0f) sink[1] = x + z.x + key + f;
}

int main() {
  long long *out; double *sink;
  cudaMallocManaged(&out, 8); cudaMalloc(&sink, 16);
  const char *names[] = {"dfma_dep", "crecip", "credux", "shfl_f64", "f2f_roundtrip", "rcp_f64"};
  for (int load = 0; load <= 3; load += 3) {
    for (int op = 0; op < 6; ++op) {
      switch (op) {
        case 0: probe<0><<<1, 512>>>(out, sink, load); break;
        case 1: probe<1><<<1, 512>>>(out, sink, load); break;
        case 2: probe<2><<<1, 512>>>(out, sink, load); break;
        case 3: probe<3><<<1, 512>>>(out, sink, load); break;
        case 4: probe<4><<<1, 512>>>(out, sink, load); break;
        case 5: probe<5><<<1, 512>>>(out, sink, load); break;
      }
      cudaDeviceSynchronize();
      printf("{\"op\":\"%s\",\"bg_dfma_warps_per_smsp\":%d,\"clk_per_iter\":%lld}\n", names[op], load, out[0]);
    }
  }
  return 0;
}
