// FP64 throughput microbenchmark for B200 (sm_100a): DFMA (vector pipe) and
// DMMA (mma.sync.m8n8k4.f64, the only FP64 tensor path on sm_100a).
// Burst: one ~50 ms launch, best of 5.  Sustained: back-to-back launches for ~4 s.
// Prints JSON lines: {"kind":..., "tflops":..., "ms":...}
#include <cstdio>
#include <cuda_runtime.h>
#include <chrono>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int CHAINS>
__global__ void dfma_kernel(double *out, long iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-9 + c;
  for (long i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.0) out[0] = s;
}

template <int CHAINS>
__global__ void dmma_kernel(double *out, long iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[CHAINS][2];
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) { c[k][0] = 0; c[k][1] = 0; }
  for (long i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < CHAINS; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.0) out[0] = s;
}

// half the warps issue DFMA chains, half issue DMMA: do the two FP64 paths share one pipe?
__global__ void mixed_kernel(double *out, long iters_f, long iters_m) {
  const int warp = threadIdx.x >> 5;
  if (warp & 1) {
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
    double c[4][2] = {};
    for (long i = 0; i < iters_m; ++i) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
    }
    double s = 0;
    for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
    if (s == 12345.0) out[0] = s;
  } else {
    double acc[8];
    for (int c = 0; c < 8; ++c) acc[c] = threadIdx.x * 1e-9 + c;
    for (long i = 0; i < iters_f; ++i) {
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[c] = fma(acc[c], 0.999999, 1e-7);
    }
    double s = 0;
    for (int c = 0; c < 8; ++c) s += acc[c];
    if (s == 12345.0) out[0] = s;
  }
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("{\"device\":\"%s\",\"sms\":%d,\"smem_per_block_optin\":%zu,\"regs_per_sm\":%d}\n",
         p.name, p.multiProcessorCount, p.sharedMemPerBlockOptin, p.regsPerMultiprocessor);
  double *out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  for (int blocks_per_sm : {2, 4, 8}) {
    int threads = 256;
    long iters = 20000;
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      dfma_kernel<8><<<sms * blocks_per_sm, threads>>>(out, iters, 0.999999, 1e-7);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double flops = 2.0 * 8 * iters * (double)threads * sms * blocks_per_sm;
    printf("{\"kind\":\"dfma_burst\",\"blocks_per_sm\":%d,\"ms\":%.3f,\"tflops\":%.3f}\n", blocks_per_sm, best, flops / best / 1e9);
  }
  for (int blocks_per_sm : {2, 4, 8}) {
    int threads = 256;
    long iters = 4000;
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      dmma_kernel<4><<<sms * blocks_per_sm, threads>>>(out, iters);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double flops = 2.0 * 256 * 4 * iters * (double)(threads / 32) * sms * blocks_per_sm;
    printf("{\"kind\":\"dmma_burst\",\"blocks_per_sm\":%d,\"ms\":%.3f,\"tflops\":%.3f}\n", blocks_per_sm, best, flops / best / 1e9);
  }
  {
    // mixed: 4 blocks/SM x 256 threads; even warps DFMA (iters_f), odd warps DMMA (iters_m)
    const int threads = 256, bps = 4;
    const long iters_f = 20000, iters_m = 4000;
    for (int mode = 0; mode < 1; ++mode) {
      float best = 1e30f;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        mixed_kernel<<<sms * bps, threads>>>(out, iters_f, iters_m);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      const double nw = (double)sms * bps * (threads / 32) / 2;  // warps of each kind
      const double fl_f = 2.0 * 8 * iters_f * 32 * nw, fl_m = 2.0 * 256 * 4 * iters_m * nw;
      printf("{\"kind\":\"mixed_dfma_dmma\",\"ms\":%.3f,\"tflops_total\":%.3f,\"tflops_dfma_part\":%.3f,\"tflops_dmma_part\":%.3f}\n",
             best, (fl_f + fl_m) / best / 1e9, fl_f / best / 1e9, fl_m / best / 1e9);
    }
  }
  // sustained: ~4 s of back-to-back launches
  for (int which = 0; which < 2; ++which) {
    int threads = 256, bps = 4;
    long iters = which == 0 ? 20000 : 4000;
    double flops1 = which == 0 ? 2.0 * 8 * iters * (double)threads * sms * bps
                               : 2.0 * 256 * 4 * iters * (double)(threads / 32) * sms * bps;
    auto t0 = std::chrono::steady_clock::now();
    int n = 0; float total = 0;
    while (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() < 4.0) {
      cudaEventRecord(e0);
      for (int k = 0; k < 10; ++k) {
        if (which == 0) dfma_kernel<8><<<sms * bps, threads>>>(out, iters, 0.999999, 1e-7);
        else dmma_kernel<4><<<sms * bps, threads>>>(out, iters);
      }
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1); total += ms; n += 10;
    }
    printf("{\"kind\":\"%s_sustained\",\"launches\":%d,\"ms_per_launch\":%.3f,\"tflops\":%.3f}\n",
           which == 0 ? "dfma" : "dmma", n, total / n, flops1 * n / total / 1e9);
  }
  return 0;
}
