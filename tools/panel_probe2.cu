// Panel-factorisation latency probe, position-tracking variant used by k_lu_blk.cu (dev tool).
// One warp factors a 48 x 8 complex panel (partial pivoting, rows never move) 16 times; optionally a second warp on
// the SAME SM sub-partition (warp 4 of the block) streams independent DMMAs to measure FP64-pipe contention.
//   VAR 0: kernel algorithm (key with position, speculative reciprocal, smem broadcast, full-width update)
//   VAR 1: + in-panel lookahead (column j+1 updated and its key formed before the other columns)
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2307_05590_b200/csrc/podp_common.cuh"
using namespace podp;

__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int VAR>
__global__ void probe(double2 *g, long long *out, int contend) {
  constexpr int NB = 8, MS = 2, R = 48, LDA = 57;
  __shared__ double2 A[R * LDA];
  __shared__ double2 sRowP[2 * NB], sRinv[R];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned FULL = 0xffffffffu;
  __shared__ volatile int done;
  if (threadIdx.x == 0) done = 0;
  for (int e = threadIdx.x; e < R * LDA; e += blockDim.x) A[e] = g[e];
  __syncthreads();
  if (wid != 0) {
    if (!contend || wid != 4) return;
    double c[8][2] = {};
    double av = 1.0 + lane * 1e-3, bv = 1.0 - lane * 1e-3;
    for (int it = 0; it < (1 << 20) && !done; ++it) {
      if (contend == 1) {
#pragma unroll
        for (int q = 0; q < 8; ++q) dmma(c[q][0], c[q][1], av, bv);
      } else if (contend == 3) {
#pragma unroll
        for (int q = 0; q < 8; ++q) dmma(c[0][0], c[0][1], av, bv);  // one dependent chain
      } else if (contend == 4) {
#pragma unroll
        for (int q = 0; q < 8; ++q) dmma(c[q & 1][0], c[q & 1][1], av, bv);  // two chains
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          c[q][0] = fma(av, bv, c[q][0]);
          c[q][1] = fma(bv, av, c[q][1]);
        }
      }
    }
    double s = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) s += c[q][0] + c[q][1];
    if (s == 12345.0) out[60] = 1;
    return;
  }
  long long t0 = clock64();
  const int kb = 0;
  for (int rep = 0; rep < 16; ++rep) {
    double2 pn[MS][NB];
    int pos[MS];
#pragma unroll
    for (int m = 0; m < MS; ++m) {
      const int i = kb + lane + 32 * m;
      pos[m] = i < R ? i : 1 << 20;
#pragma unroll
      for (int c = 0; c < NB; ++c) pn[m][c] = (i < R) ? A[i * LDA + kb + c] : make_double2(0.0, 0.0);
    }
    unsigned key = 0u;
    double2 cand = pn[0][0];
#pragma unroll
    for (int m = 0; m < MS; ++m) {
      const unsigned kk = (mag_key_hi(pn[m][0]) & 0xFFFFFF80u) | (unsigned)(127 - pos[m]);
      if (pos[m] < R && kk > key) { key = kk; cand = pn[m][0]; }
    }
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      const int kr = kb + j;
      if (VAR != 1 && j > 0) {
        key = 0u;
        cand = pn[0][j];
#pragma unroll
        for (int m = 0; m < MS; ++m) {
          const unsigned kk = (mag_key_hi(pn[m][j]) & 0xFFFFFF80u) | (unsigned)(127 - pos[m]);
          if (pos[m] >= kr && pos[m] < R && kk > key) { key = kk; cand = pn[m][j]; }
        }
      }
      const double2 rc_mine = (VAR == 3 || VAR == 4) ? cand : crecip_fast(cand);
      const unsigned best = (VAR == 2 || VAR == 4) ? (unsigned)(127 - kr) : __reduce_max_sync(FULL, key);
      const int p = 127 - (int)(best & 127u);
      bool mine[MS];
#pragma unroll
      for (int m = 0; m < MS; ++m) {
        mine[m] = pos[m] == p;
        if (mine[m]) {
#pragma unroll
          for (int c = j + 1; c < NB; ++c) sRowP[c] = pn[m][c];
          sRowP[NB] = rc_mine;
        }
      }
      __syncwarp();
      const double2 rc = sRowP[NB];
      double2 u[NB];
#pragma unroll
      for (int c = j + 1; c < NB; ++c) u[c] = sRowP[c];
#pragma unroll
      for (int m = 0; m < MS; ++m) pos[m] = mine[m] ? kr : (pos[m] == kr ? p : pos[m]);
      if (lane == 0) sRinv[kr] = rc;
      double2 l[MS];
#pragma unroll
      for (int m = 0; m < MS; ++m) {
        const bool act = pos[m] > kr && pos[m] < R;
        l[m] = act ? cmul(pn[m][j], rc) : make_double2(0.0, 0.0);
        if (act) pn[m][j] = l[m];
      }
      if (VAR == 1 && j + 1 < NB) {
        // next column first, then its key, then the rest
#pragma unroll
        for (int m = 0; m < MS; ++m) pn[m][j + 1] = cfms(l[m], u[j + 1], pn[m][j + 1]);
        key = 0u;
        cand = pn[0][j + 1];
#pragma unroll
        for (int m = 0; m < MS; ++m) {
          const unsigned kk = (mag_key_hi(pn[m][j + 1]) & 0xFFFFFF80u) | (unsigned)(127 - pos[m]);
          if (pos[m] >= kr + 1 && pos[m] < R && kk > key) { key = kk; cand = pn[m][j + 1]; }
        }
#pragma unroll
        for (int c = j + 2; c < NB; ++c)
#pragma unroll
          for (int m = 0; m < MS; ++m) pn[m][c] = cfms(l[m], u[c], pn[m][c]);
      } else {
#pragma unroll
        for (int c = j + 1; c < NB; ++c)
#pragma unroll
          for (int m = 0; m < MS; ++m) pn[m][c] = cfms(l[m], u[c], pn[m][c]);
      }
      __syncwarp();
    }
#pragma unroll
    for (int m = 0; m < MS; ++m)
      if (pos[m] < R)
#pragma unroll
        for (int c = 0; c < NB; ++c) A[pos[m] * LDA + kb + c] = pn[m][c];
    __syncwarp();
  }
  long long t1 = clock64();
  if (lane == 0) { out[VAR * 5 + contend] = (t1 - t0) / 16; done = 1; }
  for (int e = lane; e < R * LDA; e += 32) g[e] = A[e];
}

int main() {
  double2 *g; long long *out;
  cudaMalloc(&g, 48 * 57 * 16); cudaMallocManaged(&out, 64 * 8); cudaMemset(out, 0, 64 * 8);
  static double2 h[48 * 57];
  for (int i = 0; i < 48 * 57; ++i) h[i] = make_double2(1.0 + (i * 7919 % 97) * 0.01, (i * 104729 % 89) * 0.01);
  for (int i = 0; i < 48; ++i) h[i * 57 + (i % 8)] = make_double2(100.0 + i, 0.0);
  for (int contend = 0; contend < 5; ++contend) {
    for (int v = 0; v < 5; ++v) {
      if (contend && v > 1) continue;
      cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice);
      if (v == 0) probe<0><<<1, 160>>>(g, out, contend);
      if (v == 1) probe<1><<<1, 160>>>(g, out, contend);
      if (v == 2) probe<2><<<1, 160>>>(g, out, contend);
      if (v == 3) probe<3><<<1, 160>>>(g, out, contend);
      if (v == 4) probe<4><<<1, 160>>>(g, out, contend);
      cudaError_t e = cudaDeviceSynchronize();
      printf("{\"var\":%d,\"contend\":%d,\"clk_per_panel\":%lld,\"clk_per_column\":%lld,\"err\":\"%s\"}\n", v, contend,
             out[v * 5 + contend], out[v * 5 + contend] / 8, cudaGetErrorString(e));
    }
  }
  return 0;
}
