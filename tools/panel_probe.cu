// Panel-factorisation latency probe (dev tool): one warp factors a 48 x 8 complex panel in registers with partial
// pivoting, repeatedly; variants isolate the cost of each part of the per-column chain.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2307_05590_b200/csrc/podp_common.cuh"
using namespace podp;

template <int VAR>
__global__ void panel_probe(double2 *g, long long *out) {
  constexpr int NB = 8, MS = 2, R = 48, LDA = 60;
  __shared__ double2 A[R * LDA];
  __shared__ double2 sRowK[NB], sRowP[NB], sRinv[R];
  __shared__ int sPiv[R];
  const int lane = threadIdx.x;
  for (int e = lane; e < R * LDA; e += 32) A[e] = g[e];
  __syncwarp();
  long long t0 = clock64();
  const int kb = 0;
  for (int rep = 0; rep < 16; ++rep) {
    double2 pn[MS][NB];
#pragma unroll
    for (int m = 0; m < MS; ++m) {
      const int i = kb + lane + 32 * m;
#pragma unroll
      for (int c = 0; c < NB; ++c) pn[m][c] = (i < R) ? A[i * LDA + kb + c] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      const int kr = kb + j;
      int p = kr;
      if (VAR != 2) {
        unsigned key = 0u;
#pragma unroll
        for (int m = 0; m < MS; ++m) {
          const int i = kb + lane + 32 * m;
          const unsigned kk = (mag_key_hi(pn[m][j]) & 0xFFFFFF80u) | (unsigned)(127 - i);
          if (i >= kr && i < R && kk > key) key = kk;
        }
        const unsigned best = __reduce_max_sync(0xffffffffu, key);
        p = 127 - (int)(best & 127u);
      }
      const int lp = (p - kb) & 31, mp = (p - kb) >> 5;
      if (lane == lp) {
#pragma unroll
        for (int m = 0; m < MS; ++m)
          if (m == mp) {
#pragma unroll
            for (int c = 0; c < NB; ++c) sRowP[c] = pn[m][c];
          }
      }
      if (VAR == 0 && lane == j && p != kr) {
#pragma unroll
        for (int c = 0; c < NB; ++c) sRowK[c] = pn[0][c];
      }
      if (lane == 0) sPiv[kr] = p;
      __syncwarp();
      const double2 pv = sRowP[j];
      double2 u[NB];
#pragma unroll
      for (int c = j + 1; c < NB; ++c) u[c] = sRowP[c];
      if (VAR == 0 && p != kr) {
        if (lane == lp) {
#pragma unroll
          for (int m = 0; m < MS; ++m)
            if (m == mp) {
#pragma unroll
              for (int c = 0; c < NB; ++c) pn[m][c] = sRowK[c];
            }
        }
        if (lane == j) {
#pragma unroll
          for (int c = 0; c < NB; ++c) pn[0][c] = sRowP[c];
        }
      }
      const double2 rc = crecip_fast(pv);
      if (lane == 0) sRinv[kr] = rc;
      double2 l[MS];
#pragma unroll
      for (int m = 0; m < MS; ++m) {
        const int i = kb + lane + 32 * m;
        const bool act = i > kr && i < R;
        l[m] = act ? cmul(pn[m][j], rc) : make_double2(0.0, 0.0);
        if (act) pn[m][j] = l[m];
      }
#pragma unroll
      for (int c = j + 1; c < NB; ++c) {
#pragma unroll
        for (int m = 0; m < MS; ++m) pn[m][c] = cfms(l[m], u[c], pn[m][c]);
      }
      __syncwarp();
    }
#pragma unroll
    for (int m = 0; m < MS; ++m) {
      const int i = kb + lane + 32 * m;
      if (i < R) {
#pragma unroll
        for (int c = 0; c < NB; ++c) A[i * LDA + kb + c] = pn[m][c];
      }
    }
    __syncwarp();
  }
  long long t1 = clock64();
  if (lane == 0) out[VAR] = (t1 - t0) / 16;
  for (int e = lane; e < R * LDA; e += 32) g[e] = A[e];
}

int main() {
  double2 *g; long long *out;
  cudaMalloc(&g, 48 * 60 * 16); cudaMallocManaged(&out, 64);
  double2 h[48 * 60];
  for (int i = 0; i < 48 * 60; ++i) h[i] = make_double2(1.0 + (i * 7919 % 97) * 0.01, (i * 104729 % 89) * 0.01);
  for (int i = 0; i < 48; ++i) h[i * 60 + (i % 8)] = make_double2(100.0 + i, 0.0);
  const char *names[] = {"full(pivot+swap)", "pivot_no_swap", "no_pivot"};
  for (int v = 0; v < 3; ++v) {
    cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice);
    if (v == 0) panel_probe<0><<<1, 32>>>(g, out);
    if (v == 1) panel_probe<1><<<1, 32>>>(g, out);
    if (v == 2) panel_probe<2><<<1, 32>>>(g, out);
    cudaDeviceSynchronize();
    printf("{\"panel\":\"%s\",\"clk_per_panel\":%lld,\"clk_per_column\":%lld}\n", names[v], out[v], out[v] / 8);
  }
  return 0;
}
