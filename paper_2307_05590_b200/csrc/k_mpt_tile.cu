// K3: MPT quadratic forms + error certificate, rows a4-a6 of SURVEY 8(a): R (eqn:podprealmpt), I
// (eqn:podpimagmpt) and Delta (lemma:certificate, in the re-associated form of SURVEY
// Appendix A.2: X_ij = c_ij + l_i p_j + conj(l_j p_i) + p_i^H Q(omega) p_j).
//
//   For every frequency and every pair i <= j:  Re(p_i^H K_R p_j), Re(p_i^H M p_j), Re(p_i^H Q(omega) p_j) with
//   Q = G_KK + s J + s^2 G_MM formed on the fly (Horner, 4 DFMA per element), plus Re(l_i p_j), Re(h_i p_j).
//
// Layout.  Operator-stationary: the five r x r operators (K_R, M, G_KK, J, G_MM) live in shared memory (row
// blocks of RB rows when they do not fit).  A warp owns 4 frequencies; lane = 8*f + s holds the b-slice
// {b = s + 8t} of its frequency's P (3 columns) in registers.  For each operator row a, the lane forms its partial
// y_j[a] = sum_{b in slice} Op[a][b] p_j[b] (all 8 lanes of a frequency read the same 8 consecutive operator
// entries: one conflict-free wavefront per load) and immediately contracts it with conj(p_i[a]) into 18 running
// sums; the 8 partial sums of a frequency are reduced by shuffles once per tile.  FP64 throughout.
#include "podp_common.cuh"

namespace podp {

// sizes the paired A/B kernel is instantiated for
#ifndef PODP_MPT_PAIR_SIZES
#define PODP_MPT_PAIR_SIZES PODP_MP(48)
#endif

namespace mpttile {

constexpr int WARPS = 8;
constexpr int SMEM_BUDGET = 200 * 1024;

template <int R>
struct Cfg {
  static constexpr int SL = R <= 64 ? 8 : 16;    // b-slices (lanes) per frequency
  static constexpr int FPW = 32 / SL;             // frequencies per warp
  static constexpr int TILE = WARPS * FPW;        // frequencies per CTA tile
  static constexpr int NBL = (R + SL - 1) / SL;  // b's per lane
  static constexpr int LD = R;                    // row stride (complex); 8 consecutive b's = 128 B
  static constexpr int RB_MAX = SMEM_BUDGET / (5 * R * 16);
  static constexpr int RB = RB_MAX >= R ? R : RB_MAX;  // rows per operator block
  static constexpr int NBLK = (R + RB - 1) / RB;
  static constexpr size_t BYTES = (size_t)5 * RB * LD * sizeof(double2);
};

}  // namespace mpttile

// Epilogue of one frequency: R, I (eqn:podprealmpt / eqn:podpimagmpt) and the certificate
// from the reduced sums, written as 48-byte output rows.
__device__ __forceinline__ void mpt_epilogue(const EvalArgs &a, const double *op, double w, double nu, int64_t t,
                                             const double (&qK)[6], const double (&qM)[6], const double (&qQ)[6],
                                             const double (&lp)[9], const double (&hp)[9]) {
  const double nanv = __longlong_as_double(0x7ff8000000000000ll);
  double T1[6], I[6], D[6];
  bool ok = isfinite(w);
#pragma unroll
  for (int e = 0; e < 6; ++e) ok &= isfinite(qK[e]) && isfinite(qM[e]) && isfinite(qQ[e]);
#pragma unroll
  for (int e = 0; e < 9; ++e) ok &= isfinite(lp[e]) && isfinite(hp[e]);
  if (!ok) {
#pragma unroll
    for (int e = 0; e < 6; ++e) T1[e] = I[e] = D[e] = nanv;
  } else {
    // epilogue: R, I (eqn:podprealmpt / eqn:podpimagmpt) and the certificate from the
    // reduced sums; c_ij(omega) = d^T G_{b_i b_j} d with d = (1, omega)
    const double *sc = op + a.L.scal;
    const double alpha = sc[SC_ALPHA], alb = sc[SC_ALPHA_LB];
    const double a3 = alpha * alpha * alpha;
    const double2 *Gbb = reinterpret_cast<const double2 *>(op + a.L.Gbb);
    double ReX[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const double g00 = Gbb[(2 * i) * 6 + 2 * j].x, g01 = Gbb[(2 * i) * 6 + 2 * j + 1].x;
        const double g10 = Gbb[(2 * i + 1) * 6 + 2 * j].x, g11 = Gbb[(2 * i + 1) * 6 + 2 * j + 1].x;
        const double c = g00 + w * (g01 + g10) + w * w * g11;
        ReX[i * 3 + j] = c + lp[i * 3 + j] + lp[j * 3 + i];
      }
    double n[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const double x = ReX[i * 3 + i] + qQ[i];
      n[i] = x > 0.0 ? x : 0.0;
    }
    const bool outR = a.flags & PODP_FLAG_OUT_R;
#pragma unroll
    for (int e = 0; e < 6; ++e) {
      const int i = e < 3 ? e : (e < 5 ? 0 : 1);
      const int j = e < 3 ? e : (e == 3 ? 1 : 2);
      const double Rv = -(a3 / 4.0) * qK[e];
      T1[e] = outR ? Rv : sc[SC_N0 + 3 * i + j] + Rv;
      I[e] = (w * a3 / 4.0) * (sc[SC_S + 3 * i + j] + nu * qM[e] + hp[i * 3 + j] + hp[j * 3 + i]);
      double mij = 0.0;
      if (i != j) {
        const double x = n[i] + n[j] - 2.0 * (ReX[i * 3 + j] + qQ[e]);
        mij = x > 0.0 ? x : 0.0;
      }
      D[e] = a3 / (8.0 * alb) * (n[i] + n[j] + mij);
    }
  }
  // 48-byte output rows: three 16-byte stores per quantity when the caller's arrays are 16-byte aligned (the
  // row offset t * 48 keeps that alignment), else six 8-byte stores
  double *T1p = a.T1 + (size_t)t * 6, *Ip = a.I + (size_t)t * 6, *Dp = a.Delta + (size_t)t * 6;
  if (((reinterpret_cast<uintptr_t>(a.T1) | reinterpret_cast<uintptr_t>(a.I) | reinterpret_cast<uintptr_t>(a.Delta)) &
       15) == 0) {
#pragma unroll
    for (int h = 0; h < 3; ++h) {
      reinterpret_cast<double2 *>(T1p)[h] = make_double2(T1[2 * h], T1[2 * h + 1]);
      reinterpret_cast<double2 *>(Ip)[h] = make_double2(I[2 * h], I[2 * h + 1]);
      reinterpret_cast<double2 *>(Dp)[h] = make_double2(D[2 * h], D[2 * h + 1]);
    }
  } else {
#pragma unroll
    for (int e = 0; e < 6; ++e) {
      T1p[e] = T1[e];
      Ip[e] = I[e];
      Dp[e] = D[e];
    }
  }
}

// DIAG (N3 pencil coordinates with K_R = K and M_I = M): Z^H K Z = I and Z^H M Z = Lambda, so the K_R and M_I
// quadratic forms are diagonal -- Re(y_i^H y_j) and Re(y_i^H Lambda y_j) -- and are accumulated in the slice pass;
// only Q~ = Z^H Q Z stays dense.
// BLK (N1 literal per-direction form): column i of P is nonzero only in direction block i (rows
// [a.blk_lo[i], a.blk_hi[i]), SL-aligned), so for an operator row a in block i only the pairs (i, j >= i) get a
// contribution, y_j[a] runs only over block j, and those are exactly the rectangular cross blocks K_ij^M, C_ij^M
// and the Gram blocks of eqn:podprealmpt / eqn:podpimagmpt and P:651-661.  Skipped terms are exact
// zeros, so the sums equal the dense ones bit for bit (for finite operators).
template <int R, bool DIAG, bool BLK = false>
__global__ void __launch_bounds__(mpttile::WARPS * 32, 1) mpt_tile_kernel(EvalArgs a) {
  using C = mpttile::Cfg<R>;
  constexpr int NBL = C::NBL, RB = C::RB, NBLK = C::NBLK, LD = C::LD, SL = C::SL, TILE = C::TILE, FPW = C::FPW;
  extern __shared__ double2 smem[];
  double2 *sKR = smem, *sM = sKR + RB * LD, *sGk = sM + RB * LD, *sJ = sGk + RB * LD, *sGm = sJ + RB * LD;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int fl = lane / SL, sl = lane % SL;
  const int64_t total = (int64_t)a.n_obj * a.F;
  const int64_t ntiles = (total + TILE - 1) / TILE;
  int loaded_obj = -1;
  const double nanv = __longlong_as_double(0x7ff8000000000000ll);

  // Multi-object launches take a contiguous range of tiles per CTA (operators are re-staged only where the range
  // crosses an object boundary, not on nearly every tile as with a round-robin assignment); one object: round robin.
  const bool blocked = a.n_obj > 1;
  const int64_t per_cta = (ntiles + gridDim.x - 1) / gridDim.x;
  const int64_t tile_begin = blocked ? (int64_t)blockIdx.x * per_cta : blockIdx.x;
  const int64_t tile_end = blocked ? (tile_begin + per_cta < ntiles ? tile_begin + per_cta : ntiles) : ntiles;
  const int64_t tile_step = blocked ? 1 : gridDim.x;
  for (int64_t tile = tile_begin; tile < tile_end; tile += tile_step) {
    const int64_t t0 = tile * TILE;
    int64_t t = t0 + warp * FPW + fl;  // my frequency (global evaluation index)
    const bool valid = t < total;
    if (!valid) t = total - 1;
    const int obj = (int)(t / a.F);
    const int obj0 = (int)(t0 / a.F);
    const int64_t tl = (t0 + TILE - 1 < total ? t0 + TILE - 1 : total - 1);
    const bool one_obj = obj0 == (int)(tl / a.F);  // whole tile belongs to one object
    const int64_t f = t - (int64_t)obj * a.F;
    const double *op = a.ops + (size_t)obj * a.L.stride;
    const double w = a.omega[f];
    const double nu = op[a.L.scal + SC_NU];
    const double s = w * nu;
    // my slice of P (3 columns) into registers
    const double2 *Pw = a.Pws + (size_t)t * 3 * R;
    double2 p[NBL][3];
#pragma unroll
    for (int tt = 0; tt < NBL; ++tt) {
      const int b = sl + SL * tt;
#pragma unroll
      for (int c = 0; c < 3; ++c) p[tt][c] = (b < R) ? Pw[c * R + b] : make_double2(0.0, 0.0);
    }
    double qK[6], qM[6], qQ[6], lp[9], hp[9];
#pragma unroll
    for (int e = 0; e < 6; ++e) qK[e] = qM[e] = qQ[e] = 0.0;
    if constexpr (DIAG) {
      const double *lam = op + a.L.lam;
#pragma unroll
      for (int tt = 0; tt < NBL; ++tt) {
        const int b = sl + SL * tt;
        if (b < R) {
          const double lb = lam[b];
#pragma unroll
          for (int e = 0; e < 6; ++e) {
            const int i = e < 3 ? e : (e < 5 ? 0 : 1);
            const int j = e < 3 ? e : (e == 3 ? 1 : 2);
            const double re = fma(p[tt][i].x, p[tt][j].x, p[tt][i].y * p[tt][j].y);
            qK[e] += re;
            qM[e] = fma(lb, re, qM[e]);
          }
        }
      }
    }
    // linear terms over my slice: Re(l_i[b] p_j[b]), Re(h_i[b] p_j[b])
    {
      const double2 *GbK = reinterpret_cast<const double2 *>(op + a.L.GbK);
      const double2 *GbM = reinterpret_cast<const double2 *>(op + a.L.GbM);
      const double2 *H = reinterpret_cast<const double2 *>(op + a.L.H);
#pragma unroll
      for (int e = 0; e < 9; ++e) lp[e] = hp[e] = 0.0;
#pragma unroll
      for (int tt = 0; tt < NBL; ++tt) {
        const int b = sl + SL * tt;
        if (b < R) {
#pragma unroll
          for (int i = 0; i < 3; ++i) {
            const double2 k0 = __ldg(GbK + (2 * i) * R + b), k1 = __ldg(GbK + (2 * i + 1) * R + b);
            const double2 m0 = __ldg(GbM + (2 * i) * R + b), m1 = __ldg(GbM + (2 * i + 1) * R + b);
            const double2 gk = make_double2(fma(w, k1.x, k0.x), fma(w, k1.y, k0.y));
            const double2 gm = make_double2(fma(w, m1.x, m0.x), fma(w, m1.y, m0.y));
            const double2 l = make_double2(-gk.x + s * gm.y, -gk.y - s * gm.x);
            const double2 h = __ldg(H + i * R + b);
#pragma unroll
            for (int j = 0; j < 3; ++j) {
              lp[i * 3 + j] = fma(l.x, p[tt][j].x, fma(-l.y, p[tt][j].y, lp[i * 3 + j]));
              hp[i * 3 + j] = fma(h.x, p[tt][j].x, fma(-h.y, p[tt][j].y, hp[i * 3 + j]));
            }
          }
        }
      }
    }
    // quadratic forms, operator rows in blocks
#pragma unroll 1
    for (int blk = 0; blk < NBLK; ++blk) {
      const int a0 = blk * RB, a1 = (a0 + RB < R) ? a0 + RB : R;
      const bool need_load = one_obj && (NBLK > 1 || loaded_obj != obj0);  // CTA-uniform
      if (need_load) {
        __syncthreads();
        const double *opl = a.ops + (size_t)obj0 * a.L.stride;
        const double2 *gKR = reinterpret_cast<const double2 *>(opl + a.L.KR);
        const double2 *gM = reinterpret_cast<const double2 *>(opl + a.L.MI);
        const double2 *gGk = reinterpret_cast<const double2 *>(opl + a.L.Gkk);
        const double2 *gJ = reinterpret_cast<const double2 *>(opl + a.L.J);
        const double2 *gGm = reinterpret_cast<const double2 *>(opl + a.L.Gmm);
        const int n = (a1 - a0) * R;
        for (int e = threadIdx.x; e < n; e += blockDim.x) {
          const int row = e / R, col = e - row * R;
          const int src = (a0 + row) * R + col, dst = row * LD + col;
          if constexpr (!DIAG) {
            sKR[dst] = gKR[src];
            sM[dst] = gM[src];
          }
          sGk[dst] = gGk[src];
          sJ[dst] = gJ[src];
          sGm[dst] = gGm[src];
        }
        __syncthreads();
        loaded_obj = NBLK == 1 ? obj0 : -1;
      }
      // operators for this frequency: shared-memory block (tile of one object) or global (mixed tile)
      const bool shared_ops = one_obj;
      const double2 *oKR = shared_ops ? sKR : reinterpret_cast<const double2 *>(op + a.L.KR) + a0 * R;
      const double2 *oM = shared_ops ? sM : reinterpret_cast<const double2 *>(op + a.L.MI) + a0 * R;
      const double2 *oGk = shared_ops ? sGk : reinterpret_cast<const double2 *>(op + a.L.Gkk) + a0 * R;
      const double2 *oJ = shared_ops ? sJ : reinterpret_cast<const double2 *>(op + a.L.J) + a0 * R;
      const double2 *oGm = shared_ops ? sGm : reinterpret_cast<const double2 *>(op + a.L.Gmm) + a0 * R;
      const int ld = shared_ops ? LD : R;
      // conj(p_i[a]) of the next operator row is fetched one iteration ahead (its L1/L2 latency showed as
      // long-scoreboard stalls on the contraction at the end of each row)
      double2 pn[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) pn[c] = __ldg(Pw + c * R + a0);
#pragma unroll 1
      for (int ar = a0; ar < a1; ++ar) {
        const int row = (ar - a0) * ld;
        // BLK: block of this operator row (warp-uniform); only pairs (cb, j >= cb) receive contributions
        const int cb = BLK ? (ar < a.blk_hi[0] ? 0 : (ar < a.blk_hi[1] ? 1 : 2)) : 0;
        double2 pa[3];
        const int an = ar + 1 < a1 ? ar + 1 : ar;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          pa[c] = pn[c];
          pn[c] = __ldg(Pw + c * R + an);
        }
        double2 yK[3], yM[3], yQ[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) yK[c] = yM[c] = yQ[c] = make_double2(0.0, 0.0);
#pragma unroll
        for (int tt = 0; tt < NBL; ++tt) {
          const int b = sl + SL * tt;
          if constexpr (BLK) {
            // b-group [SL tt, SL tt + SL) lies in one block gb (blocks are SL-aligned): only column gb is nonzero
            // there, and it is needed only if gb >= cb
            const int gb = SL * tt < a.blk_hi[0] ? 0 : (SL * tt < a.blk_hi[1] ? 1 : 2);
            if (gb < cb) continue;
            const double2 gk = oGk[row + b], jj = oJ[row + b], gm = oGm[row + b];
            const double2 q = make_double2(fma(s, fma(s, gm.x, jj.x), gk.x), fma(s, fma(s, gm.y, jj.y), gk.y));
            const double2 kr = oKR[row + b], mm = oM[row + b];
            switch (gb) {
              case 0:
                yK[0] = cfma(kr, p[tt][0], yK[0]);
                yM[0] = cfma(mm, p[tt][0], yM[0]);
                yQ[0] = cfma(q, p[tt][0], yQ[0]);
                break;
              case 1:
                yK[1] = cfma(kr, p[tt][1], yK[1]);
                yM[1] = cfma(mm, p[tt][1], yM[1]);
                yQ[1] = cfma(q, p[tt][1], yQ[1]);
                break;
              default:
                yK[2] = cfma(kr, p[tt][2], yK[2]);
                yM[2] = cfma(mm, p[tt][2], yM[2]);
                yQ[2] = cfma(q, p[tt][2], yQ[2]);
                break;
            }
          } else if ((R % SL) == 0 || b < R) {
            const double2 gk = oGk[row + b], jj = oJ[row + b], gm = oGm[row + b];
            const double2 q = make_double2(fma(s, fma(s, gm.x, jj.x), gk.x), fma(s, fma(s, gm.y, jj.y), gk.y));
            if constexpr (!DIAG) {
              const double2 kr = oKR[row + b], mm = oM[row + b];
#pragma unroll
              for (int c = 0; c < 3; ++c) {
                yK[c] = cfma(kr, p[tt][c], yK[c]);
                yM[c] = cfma(mm, p[tt][c], yM[c]);
              }
            }
#pragma unroll
            for (int c = 0; c < 3; ++c) yQ[c] = cfma(q, p[tt][c], yQ[c]);
          }
        }
#pragma unroll
        for (int e = 0; e < 6; ++e) {
          const int i = e < 3 ? e : (e < 5 ? 0 : 1);
          const int j = e < 3 ? e : (e == 3 ? 1 : 2);
          if (BLK && i != cb) continue;  // conj(p_i[a]) = 0 outside block i
          if constexpr (!DIAG) {
            qK[e] = fma(pa[i].x, yK[j].x, fma(pa[i].y, yK[j].y, qK[e]));
            qM[e] = fma(pa[i].x, yM[j].x, fma(pa[i].y, yM[j].y, qM[e]));
          }
          qQ[e] = fma(pa[i].x, yQ[j].x, fma(pa[i].y, yQ[j].y, qQ[e]));
        }
      }
    }
    // reduce the SL partial sums of each frequency (lanes SL*f .. SL*f+SL-1)
#pragma unroll
    for (int o = 1; o < SL; o <<= 1) {
#pragma unroll
      for (int e = 0; e < 6; ++e) {
        qK[e] += __shfl_xor_sync(0xffffffffu, qK[e], o);
        qM[e] += __shfl_xor_sync(0xffffffffu, qM[e], o);
        qQ[e] += __shfl_xor_sync(0xffffffffu, qQ[e], o);
      }
#pragma unroll
      for (int e = 0; e < 9; ++e) {
        lp[e] += __shfl_xor_sync(0xffffffffu, lp[e], o);
        hp[e] += __shfl_xor_sync(0xffffffffu, hp[e], o);
      }
    }
    if (valid && sl == 0) {
      mpt_epilogue(a, op, w, nu, t, qK, qM, qQ, lp, hp);
    }
  }
}

// Paired A/B variant (PODP_FLAG_MPT_PAIR; one object, R <= 48, no DIAG / BLK; measured SLOWER than the kernel above,
// 1.00 vs 0.94 ms per 1e5 at r = 48: ncu shows the shared-memory pipe down from 69 % to 48 % but the FP64 pipe only
// at 70 % -- with 2 warps per SM sub-partition the kernel is bound by its dependent-DFMA issue, not by the operator
// traffic -- while it executes 13 % more flops): a lane keeps the b-slices of TWO frequencies (16 lanes per
// frequency pair, 3 b's per lane at R = 48), so every operator entry fetched from shared memory feeds two
// frequencies.  The one-frequency-per-lane kernel above reads all five operators once per frequency -- 184 KB, 1500
// shared-memory wavefronts at R = 48 (a 16-byte load costs 4 wavefronts per warp whatever the 4 frequencies of the
// warp have in common), which ncu shows at 69 % of the pipe beside 66 % FP64; here the wavefronts halve.  The per-lane
// contraction of each row's partial products is done by 16 instead of 8 lanes per frequency (executed flops
// F_alg + 26 % instead of + 13 %).  Operators are processed one after another (K_R, M_I, Q) to bound the registers.
namespace mptpair {
constexpr int WARPS = 8;
template <int R>
struct Cfg {
  static constexpr int SL = 16, NBL = (R + SL - 1) / SL, FPW = 4, TILE = WARPS * FPW;
  static constexpr size_t BYTES = (size_t)5 * R * R * sizeof(double2);
};
}  // namespace mptpair

template <int R>
__global__ void __launch_bounds__(mptpair::WARPS * 32, 1) mpt_pair_kernel(EvalArgs a) {
  using C = mptpair::Cfg<R>;
  constexpr int NBL = C::NBL, SL = C::SL, TILE = C::TILE;
  extern __shared__ double2 smem[];
  double2 *sKR = smem, *sM = sKR + R * R, *sGk = sM + R * R, *sJ = sGk + R * R, *sGm = sJ + R * R;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 4, sl = lane & 15;
  const double *op = a.ops;  // one object
  {
    const double2 *gKR = reinterpret_cast<const double2 *>(op + a.L.KR);
    const double2 *gM = reinterpret_cast<const double2 *>(op + a.L.MI);
    const double2 *gGk = reinterpret_cast<const double2 *>(op + a.L.Gkk);
    const double2 *gJ = reinterpret_cast<const double2 *>(op + a.L.J);
    const double2 *gGm = reinterpret_cast<const double2 *>(op + a.L.Gmm);
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
      sKR[e] = gKR[e];
      sM[e] = gM[e];
      sGk[e] = gGk[e];
      sJ[e] = gJ[e];
      sGm[e] = gGm[e];
    }
    __syncthreads();
  }
  const int64_t total = a.F;
  const int64_t ntiles = (total + TILE - 1) / TILE;
  const double nu = op[a.L.scal + SC_NU];
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    int64_t t[2];
    bool valid[2];
    double w[2], s[2];
    const double2 *Pw[2];
    double2 p[2][NBL][3];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      t[u] = tile * TILE + warp * C::FPW + g * 2 + u;
      valid[u] = t[u] < total;
      if (!valid[u]) t[u] = total - 1;
      w[u] = a.omega[t[u]];
      s[u] = w[u] * nu;
      Pw[u] = a.Pws + (size_t)t[u] * 3 * R;
#pragma unroll
      for (int tt = 0; tt < NBL; ++tt) {
        const int b = sl + SL * tt;
#pragma unroll
        for (int c = 0; c < 3; ++c) p[u][tt][c] = (b < R) ? Pw[u][c * R + b] : make_double2(0.0, 0.0);
      }
    }
    double qK[2][6], qM[2][6], qQ[2][6];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int e = 0; e < 6; ++e) qK[u][e] = qM[u][e] = qQ[u][e] = 0.0;
    // y_j[a] partial over my slice for one operator value per b, contracted with conj(p_i[a]) into q
    auto contract = [&](const double2 (&y)[2][3], const double2 (&pa)[2][3], double (&q)[2][6]) {
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int e = 0; e < 6; ++e) {
          const int i = e < 3 ? e : (e < 5 ? 0 : 1);
          const int j = e < 3 ? e : (e == 3 ? 1 : 2);
          q[u][e] = fma(pa[u][i].x, y[u][j].x, fma(pa[u][i].y, y[u][j].y, q[u][e]));
        }
    };
    double2 pn[2][3];  // conj(p_i[a]) operands of the next row, fetched one iteration ahead
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int c = 0; c < 3; ++c) pn[u][c] = __ldg(Pw[u] + c * R);
#pragma unroll 1
    for (int ar = 0; ar < R; ++ar) {
      const int row = ar * R;
      const int an = ar + 1 < R ? ar + 1 : ar;
      double2 pa[2][3];
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          pa[u][c] = pn[u][c];
          pn[u][c] = __ldg(Pw[u] + c * R + an);
        }
      {  // K_R
        double2 y[2][3];
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int c = 0; c < 3; ++c) y[u][c] = make_double2(0.0, 0.0);
#pragma unroll
        for (int tt = 0; tt < NBL; ++tt) {
          const int b = sl + SL * tt;
          if ((R % SL) == 0 || b < R) {
            const double2 kr = sKR[row + b];
#pragma unroll
            for (int u = 0; u < 2; ++u)
#pragma unroll
              for (int c = 0; c < 3; ++c) y[u][c] = cfma(kr, p[u][tt][c], y[u][c]);
          }
        }
        contract(y, pa, qK);
      }
      {  // M_I
        double2 y[2][3];
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int c = 0; c < 3; ++c) y[u][c] = make_double2(0.0, 0.0);
#pragma unroll
        for (int tt = 0; tt < NBL; ++tt) {
          const int b = sl + SL * tt;
          if ((R % SL) == 0 || b < R) {
            const double2 mm = sM[row + b];
#pragma unroll
            for (int u = 0; u < 2; ++u)
#pragma unroll
              for (int c = 0; c < 3; ++c) y[u][c] = cfma(mm, p[u][tt][c], y[u][c]);
          }
        }
        contract(y, pa, qM);
      }
      {  // Q(omega) = G_KK + s J + s^2 G_MM, formed per frequency (Horner)
        double2 y[2][3];
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int c = 0; c < 3; ++c) y[u][c] = make_double2(0.0, 0.0);
#pragma unroll
        for (int tt = 0; tt < NBL; ++tt) {
          const int b = sl + SL * tt;
          if ((R % SL) == 0 || b < R) {
            const double2 gk = sGk[row + b], jj = sJ[row + b], gm = sGm[row + b];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const double2 q = make_double2(fma(s[u], fma(s[u], gm.x, jj.x), gk.x), fma(s[u], fma(s[u], gm.y, jj.y), gk.y));
#pragma unroll
              for (int c = 0; c < 3; ++c) y[u][c] = cfma(q, p[u][tt][c], y[u][c]);
            }
          }
        }
        contract(y, pa, qQ);
      }
    }
    // linear terms Re(l_i[b] p_j[b]), Re(h_i[b] p_j[b]) over my slice, reduction over the 16 lanes, epilogue: one
    // frequency after the other (registers)
    const double2 *GbK = reinterpret_cast<const double2 *>(op + a.L.GbK);
    const double2 *GbM = reinterpret_cast<const double2 *>(op + a.L.GbM);
    const double2 *H = reinterpret_cast<const double2 *>(op + a.L.H);
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      double lp[9], hp[9];
#pragma unroll
      for (int e = 0; e < 9; ++e) lp[e] = hp[e] = 0.0;
#pragma unroll
      for (int tt = 0; tt < NBL; ++tt) {
        const int b = sl + SL * tt;
        if (b < R) {
#pragma unroll
          for (int i = 0; i < 3; ++i) {
            const double2 k0 = __ldg(GbK + (2 * i) * R + b), k1 = __ldg(GbK + (2 * i + 1) * R + b);
            const double2 m0 = __ldg(GbM + (2 * i) * R + b), m1 = __ldg(GbM + (2 * i + 1) * R + b);
            const double2 gk = make_double2(fma(w[u], k1.x, k0.x), fma(w[u], k1.y, k0.y));
            const double2 gm = make_double2(fma(w[u], m1.x, m0.x), fma(w[u], m1.y, m0.y));
            const double2 l = make_double2(-gk.x + s[u] * gm.y, -gk.y - s[u] * gm.x);
            const double2 h = __ldg(H + i * R + b);
#pragma unroll
            for (int j = 0; j < 3; ++j) {
              lp[i * 3 + j] = fma(l.x, p[u][tt][j].x, fma(-l.y, p[u][tt][j].y, lp[i * 3 + j]));
              hp[i * 3 + j] = fma(h.x, p[u][tt][j].x, fma(-h.y, p[u][tt][j].y, hp[i * 3 + j]));
            }
          }
        }
      }
#pragma unroll
      for (int o = 1; o < SL; o <<= 1) {
#pragma unroll
        for (int e = 0; e < 6; ++e) {
          qK[u][e] += __shfl_xor_sync(0xffffffffu, qK[u][e], o);
          qM[u][e] += __shfl_xor_sync(0xffffffffu, qM[u][e], o);
          qQ[u][e] += __shfl_xor_sync(0xffffffffu, qQ[u][e], o);
        }
#pragma unroll
        for (int e = 0; e < 9; ++e) {
          lp[e] += __shfl_xor_sync(0xffffffffu, lp[e], o);
          hp[e] += __shfl_xor_sync(0xffffffffu, hp[e], o);
        }
      }
      if (valid[u] && sl == 0) mpt_epilogue(a, op, w[u], nu, t[u], qK[u], qM[u], qQ[u], lp, hp);
    }
  }
}

template <int R>
static cudaError_t launch_mpt_pair_t(const EvalArgs &a, cudaStream_t s) {
  using C = mptpair::Cfg<R>;
  auto kern = mpt_pair_kernel<R>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::BYTES);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t blocks = (a.F + C::TILE - 1) / C::TILE;
  if (blocks > sms) blocks = sms;
  kern<<<(unsigned)blocks, mptpair::WARPS * 32, C::BYTES, s>>>(a);
  return cudaGetLastError();
}

template <int R>
static cudaError_t launch_mpt_tile_t(const EvalArgs &a, cudaStream_t s, bool diag) {
  using C = mpttile::Cfg<R>;
  auto kern = a.blk_hi[0] > 0 ? mpt_tile_kernel<R, false, true>
                              : (diag ? mpt_tile_kernel<R, true> : mpt_tile_kernel<R, false>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::BYTES);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t total = (int64_t)a.n_obj * a.F;
  int64_t blocks = (total + C::TILE - 1) / C::TILE;
  if (blocks > sms) blocks = sms;
  kern<<<(unsigned)blocks, mpttile::WARPS * 32, C::BYTES, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_mpt_tile(const EvalArgs &a, cudaStream_t s, bool diag) {
  // A/B variant (PODP_FLAG_MPT_PAIR; one object, dense operators, R in PODP_MPT_PAIR_SIZES): two frequencies per lane
  if (!diag && a.blk_hi[0] <= 0 && a.n_obj == 1 && (a.flags & PODP_FLAG_MPT_PAIR)) {
    switch (a.L.R) {
#define PODP_MP(R) \
      case R: return launch_mpt_pair_t<R>(a, s);
      PODP_MPT_PAIR_SIZES
#undef PODP_MP
      default: break;
    }
  }
  switch (a.L.R) {
#define PODP_MT(R) \
    case R: return launch_mpt_tile_t<R>(a, s, diag);
    PODP_MT(8) PODP_MT(16) PODP_MT(24) PODP_MT(32) PODP_MT(40) PODP_MT(48) PODP_MT(56) PODP_MT(64)
    PODP_MT(72) PODP_MT(80) PODP_MT(88) PODP_MT(96) PODP_MT(104) PODP_MT(112) PODP_MT(120) PODP_MT(128)
#undef PODP_MT
    default: return cudaErrorNotSupported;
  }
}

}  // namespace podp
