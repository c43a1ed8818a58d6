// Task functions shared by the two LU kernels (k_lu_blk.cu lock-step, k_lu_dyn.cu dynamically scheduled): panel
// factorisation with partial pivoting F(b), tile-column update U(b, c), in-place inverse of a diagonal block.
//   A(omega) = K + i omega nu M,  P = A^{-1} B  (eqn:ReducedA); [A | B] in shared memory, complex double2.
#pragma once
#include "podp_common.cuh"

namespace podp {
namespace ludyn {

__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}
// select without letting the compiler turn a slot choice into a dynamically indexed (local-memory) array
__device__ __forceinline__ double selp(bool p, double a, double b) {
  double r;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %3, 0;\n\tselp.f64 %0, %1, %2, q;\n\t}" : "=d"(r) : "d"(a), "d"(b), "r"((unsigned)p));
  return r;
}
__device__ __forceinline__ double2 shfl2(double2 v, int src) {
  return make_double2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}


// F: factor the panel at rows/cols kb.. (8 columns, rows kb..R-1) in registers; MS = row slots per lane needed for
// the R - kb panel rows.  Rows never move: each lane tracks the current position of its rows (LAPACK interchange
// semantics); the pivot search key carries the row's slot id (lowest id on ties); the pivot row is broadcast through
// an 8-entry shared scratch row.  Returns the first zero-pivot info (0 if none).
template <int R, int LDA, int MS>
__device__ __forceinline__ int factor_panel(double2 *A, double2 *sRinv, int *sOrig, int *sDst, double2 *sRow, int kb,
                                            int lane) {
  constexpr int NB = 8;
  const unsigned FULL = 0xffffffffu;
  double2 pn[MS][NB];
  int pos[MS];
#pragma unroll
  for (int m = 0; m < MS; ++m) {
    const int i = kb + lane + 32 * m;
    pos[m] = i < R ? i : (1 << 20);
#pragma unroll
    for (int c = 0; c < NB; ++c) pn[m][c] = (i < R) ? A[i * LDA + kb + c] : make_double2(0.0, 0.0);
  }
  int info = 0;
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    const int kr = kb + j;
    unsigned key = 0u;
#pragma unroll
    for (int m = 0; m < MS; ++m) {
      const unsigned kk = (mag_key_hi(pn[m][j]) & 0xFFFFFF80u) | (unsigned)(127 - (32 * m + lane));
      if (pos[m] >= kr && pos[m] < R && kk > key) key = kk;
    }
    const unsigned best = __reduce_max_sync(FULL, key);
    if ((best >> 7) == 0u) {  // exactly zero column (LAPACK getrf info = k+1); no interchange, no elimination
      if (info == 0) info = kr + 1;
      if (lane == 0) sRinv[kr] = make_double2(0.0, 0.0);
      continue;
    }
    const int id = 127 - (int)(best & 127u);
    const int src = id & 31, ms = id >> 5;  // warp-uniform: lane and slot holding the pivot row
    int p = 0;
    double2 pv, u[NB];
    if constexpr (MS == 1) {
      // one row slot: the pivot row is broadcast by shuffles (no shared-memory round trip on the chain)
      pv = shfl2(pn[0][j], src);
#pragma unroll
      for (int c = j + 1; c < NB; ++c) u[c] = shfl2(pn[0][c], src);
      p = __shfl_sync(FULL, pos[0], src);
    } else {
#pragma unroll
      for (int m = 0; m < MS; ++m) {
        if (m == ms && lane == src) {
#pragma unroll
          for (int c = j; c < NB; ++c) sRow[c] = pn[m][c];
          sRow[NB] = make_double2(__hiloint2double(0, pos[m]), 0.0);
        }
      }
      __syncwarp();
      pv = sRow[j];
#pragma unroll
      for (int c = j + 1; c < NB; ++c) u[c] = sRow[c];
      p = __double2loint(sRow[NB].x);  // current position of the pivot row
    }
#pragma unroll
    for (int m = 0; m < MS; ++m) pos[m] = (m == ms && lane == src) ? kr : (pos[m] == kr ? p : pos[m]);
    // pivots with |p|^2 outside the normal range take the call-free scaled reciprocal (uniform branch)
    const double pd = fma(pv.x, pv.x, pv.y * pv.y);
    const double2 rc = (pd >= 1e-290 && pd <= 1e290) ? crecip_fast(pv) : crecip_scaled(pv);
    if (lane == 0) sRinv[kr] = rc;
#pragma unroll
    for (int m = 0; m < MS; ++m) {
      const bool act = pos[m] > kr && pos[m] < R;
      const double2 l = act ? cmul(pn[m][j], rc) : make_double2(0.0, 0.0);
      if (act) pn[m][j] = l;
#pragma unroll
      for (int c = j + 1; c < NB; ++c) pn[m][c] = cfms(l, u[c], pn[m][c]);
    }
    if constexpr (MS > 1) __syncwarp();  // scratch row reused by the next column
  }
  // write back (L21 multipliers, L11, U11) at the final positions and record the step's permutation
#pragma unroll
  for (int m = 0; m < MS; ++m) {
    const int o = kb + lane + 32 * m;
    if (pos[m] < R) {
#pragma unroll
      for (int c = 0; c < NB; ++c) A[pos[m] * LDA + kb + c] = pn[m][c];
      if (pos[m] < kb + NB) sOrig[pos[m]] = o;
      if (o < kb + NB) sDst[o] = pos[m];
    }
  }
  __syncwarp();
  // L11^{-1} (unit lower) replaces L11 in its slots, so every U(b, .) forms U12 = L11^{-1} (P A12) on DMMA:
  // lane c < 8 solves L11 y = e_c by forward substitution (zeros above c keep the code uniform)
  if (lane < NB) {
    const int c = lane;
    double2 x[NB];
#pragma unroll
    for (int j = 0; j < NB; ++j) x[j] = make_double2(j == c ? 1.0 : 0.0, 0.0);
#pragma unroll
    for (int j = 1; j < NB; ++j) {
      double2 acc = make_double2(0.0, 0.0);
#pragma unroll
      for (int tt = 0; tt < j; ++tt) acc = cfma(A[(kb + j) * LDA + kb + tt], x[tt], acc);
      if (j > c) x[j] = make_double2(-acc.x, -acc.y);
    }
#pragma unroll
    for (int j = 1; j < NB; ++j)
      if (j > c) A[(kb + j) * LDA + kb + c] = x[j];
  }
  return info;
}

// Dinv: the inverse of the upper-triangular diagonal block U11 of a panel replaces U11 in place (its slots are dead
// once the panel is factored: trailing updates use L11^{-1}, L21 and U12 only).  Column c of the inverse comes from
// back substitution with 1/U_kk from sRinv; every lane loads its U11 entries before any lane of the warp writes.
// Tasks: lane -> (block kb0 + 8 (lane / 8), column lane % 8) for the nblk <= 4 blocks handled in one call.
template <int LDA>
__device__ __forceinline__ void invert_diag(double2 *A, const double2 *sRinv, int kb0, int nblk, int lane) {
  constexpr int NB = 8;
  double2 x[NB];
  const bool act = lane < NB * nblk;
  const int kb = kb0 + NB * (lane >> 3), c = lane & 7;
  if (act) {
    double2 u[NB][NB];
#pragma unroll
    for (int j = 0; j < NB; ++j)
#pragma unroll
      for (int t = j + 1; t < NB; ++t) u[j][t] = A[(kb + j) * LDA + kb + t];
#pragma unroll
    for (int j = NB - 1; j >= 0; --j) {
      const double2 rj = sRinv[kb + j];
      double2 acc = make_double2(0.0, 0.0);
#pragma unroll
      for (int t = j + 1; t < NB; ++t) acc = cfma(u[j][t], x[t], acc);
      x[j] = j == c ? rj : (j < c ? cmul(make_double2(-acc.x, -acc.y), rj) : make_double2(0.0, 0.0));
    }
  }
  __syncwarp();
  if (act) {
#pragma unroll
    for (int j = 0; j < NB; ++j)
      if (j <= c) A[(kb + j) * LDA + kb + c] = x[j];
  }
  __syncwarp();
}

// U: apply the panel at kb to the tile-column at col0 (NRT = row tiles below the panel, compile-time).
// The tile-column is addressed through Ct (its column 0) with row stride LDC: Ct = A + col0, LDC = LDA for a
// column in shared memory, or the group's L2-resident right-hand-side tile (LDC = 8) in the RG mode.
template <int R, int LDA, int NRT, int LDC>
__device__ __forceinline__ void update_tile_col(double2 *A, double2 *Ct, const int *sOrig, const int *sDst, int kb,
                                                int lane) {
  constexpr int NB = 8;
  // (1) permutation in one pass and U12 = L11^{-1} (P A12) on DMMA: the B-fragments of P A12 are read straight
  //     from the pivot rows' pre-step locations; lanes (row j = lane / 4, two columns) move the displaced rows out.
  {
    const int arow = lane >> 2, acol = lane & 3;
    const int bk = lane & 3, bcol = lane >> 2;
    const int crow = lane >> 2, ccol = 2 * (lane & 3);
    const double2 x0 = Ct[sOrig[kb + bk] * LDC + bcol], x1 = Ct[sOrig[kb + 4 + bk] * LDC + bcol];
    const int dst = sDst[kb + crow];
    const double2 o0 = Ct[(kb + crow) * LDC + ccol], o1 = Ct[(kb + crow) * LDC + ccol + 1];
    const double2 one = make_double2(1.0, 0.0), zero = make_double2(0.0, 0.0);
    const double2 v0 = arow > acol ? A[(kb + arow) * LDA + kb + acol] : (arow == acol ? one : zero);
    const double2 v1 = arow > acol + 4 ? A[(kb + arow) * LDA + kb + acol + 4] : (arow == acol + 4 ? one : zero);
    __syncwarp();
    if (dst >= kb + NB) {
      Ct[dst * LDC + ccol] = o0;
      Ct[dst * LDC + ccol + 1] = o1;
    }
    double er0 = 0.0, er1 = 0.0, ei0 = 0.0, ei1 = 0.0;
    dmma(er0, er1, v0.x, x0.x);
    dmma(ei0, ei1, v0.x, x0.y);
    dmma(er0, er1, -v0.y, x0.y);
    dmma(ei0, ei1, v0.y, x0.x);
    dmma(er0, er1, v1.x, x1.x);
    dmma(ei0, ei1, v1.x, x1.y);
    dmma(er0, er1, -v1.y, x1.y);
    dmma(ei0, ei1, v1.y, x1.x);
    Ct[(kb + crow) * LDC + ccol] = make_double2(er0, ei0);
    Ct[(kb + crow) * LDC + ccol + 1] = make_double2(er1, ei1);
  }
  __syncwarp();
  if constexpr (NRT > 0) {
    // (2) A22[:, tile] -= L21 U12[:, tile]: all fragment loads of a chunk of row tiles before its DMMAs
    constexpr int CH = NRT < 5 ? NRT : 5;
    const int arow = lane >> 2, acol = lane & 3;
    const int bk = lane & 3, bcol = lane >> 2;
    const int crow = lane >> 2, ccol = 2 * (lane & 3);
    const double2 b0 = Ct[(kb + bk) * LDC + bcol], b1 = Ct[(kb + 4 + bk) * LDC + bcol];
#pragma unroll
    for (int t0 = 0; t0 < NRT; t0 += CH) {
      double2 a0[CH], a1[CH], c0[CH], c1[CH];
#pragma unroll
      for (int q = 0; q < CH; ++q) {
        if (t0 + q < NRT) {
          const int tr = kb + NB + 8 * (t0 + q);
          a0[q] = A[(tr + arow) * LDA + kb + acol];
          a1[q] = A[(tr + arow) * LDA + kb + 4 + acol];
          c0[q] = Ct[(tr + crow) * LDC + ccol];
          c1[q] = Ct[(tr + crow) * LDC + ccol + 1];
        }
      }
#pragma unroll
      for (int q = 0; q < CH; ++q) {
        if (t0 + q < NRT) {
          double cr0 = c0[q].x, cr1 = c1[q].x, ci0 = c0[q].y, ci1 = c1[q].y;
          // C -= A B (complex): C_re += (-A_re) B_re + A_im B_im ; C_im += (-A_re) B_im + (-A_im) B_re
          dmma(cr0, cr1, -a0[q].x, b0.x);
          dmma(ci0, ci1, -a0[q].x, b0.y);
          dmma(cr0, cr1, a0[q].y, b0.y);
          dmma(ci0, ci1, -a0[q].y, b0.x);
          dmma(cr0, cr1, -a1[q].x, b1.x);
          dmma(ci0, ci1, -a1[q].x, b1.y);
          dmma(cr0, cr1, a1[q].y, b1.y);
          dmma(ci0, ci1, -a1[q].y, b1.x);
          c0[q] = make_double2(cr0, ci0);
          c1[q] = make_double2(cr1, ci1);
        }
      }
#pragma unroll
      for (int q = 0; q < CH; ++q) {
        if (t0 + q < NRT) {
          const int tr = kb + NB + 8 * (t0 + q);
          Ct[(tr + crow) * LDC + ccol] = c0[q];
          Ct[(tr + crow) * LDC + ccol + 1] = c1[q];
        }
      }
    }
  }
  __syncwarp();
}

template <int R, int LDA, int LDC, int N = R / 8 - 1>
__device__ __forceinline__ void update_dispatch(double2 *A, double2 *Ct, const int *sOrig, const int *sDst, int b,
                                                int lane) {
  // NRT = R/8 - 1 - b: one instantiation per panel index keeps every loop bound and offset compile-time
  if (R / 8 - 1 - b == N) {
    update_tile_col<R, LDA, N, LDC>(A, Ct, sOrig, sDst, b * 8, lane);
  } else if constexpr (N > 0) {
    update_dispatch<R, LDA, LDC, N - 1>(A, Ct, sOrig, sDst, b, lane);
  }
}

// C -> B re-layout of an 8x8 complex tile by shuffles (C: lane holds row lane/4, columns 2(lane%4), +1; B: lane holds
// rows lane%4 and lane%4 + 4 of column lane/4).
__device__ __forceinline__ void c_to_b(double2 c0, double2 c1, int lane, double2 &b0, double2 &b1) {
  const unsigned FULL = 0xffffffffu;
  const bool odd = (lane >> 2) & 1;
  const int s0 = 4 * (lane & 3) + (lane >> 3), s1 = s0 + 16;
  double2 u0, u1, w0, w1;
  u0 = shfl2(c0, s0);
  u1 = shfl2(c1, s0);
  w0 = shfl2(c0, s1);
  w1 = shfl2(c1, s1);
  (void)FULL;
  b0 = odd ? u1 : u0;
  b1 = odd ? w1 : w0;
}

}  // namespace ludyn
}  // namespace podp
