// K3: MPT quadratic-form assembler + error-certificate evaluator, rows a4-a6 of SURVEY 8(a).
//   R_ij = -(alpha^3/4) Re(p_i^H K_R p_j)                                       (eqn:podprealmpt)
//   I_ij = (omega alpha^3/4)(S_ij + nu Re(p_i^H M p_j) + Re(h_i p_j) + Re(h_j p_i))   (eqn:podpimagmpt)
//   Re X_ij = Re c_ij + Re(l_i p_j) + Re(l_j p_i) + Re(p_i^H Q p_j),  Q = G_KK + s J + s^2 G_MM, s = omega nu
//   Delta_ij = alpha^3/(8 alpha_LB)(n_i + n_j + m_ij)                            (lemma:certificate)
// (re-association of w^H G w derived in SURVEY Appendix A.2; only real parts are ever needed.)
// Generic path: one warp per (object, omega), operators read through the read-only cache.
#include "podp_common.cuh"

namespace podp {

// 18 quadratic forms (6 pairs x {K_R, M, Q}) + 9 Re(l_i p_j) + 9 Re(h_i p_j) = 36 partial sums.
struct MptSums {
  double qK[6], qM[6], qQ[6];
  double lp[9], hp[9];
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Epilogue: 6 unique entries of T1 (Rt or R), I and Delta for one omega from the reduced sums.
__device__ __forceinline__ void mpt_epilogue(const double *op, const Layout &L, double w, int flags, const MptSums &m,
                                             double *T1, double *I, double *D) {
  const double *sc = op + L.scal;
  const double nu = sc[SC_NU], alpha = sc[SC_ALPHA], alb = sc[SC_ALPHA_LB];
  const double a3 = alpha * alpha * alpha;
  const double2 *Gbb = reinterpret_cast<const double2 *>(op + L.Gbb);
  double ReX[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      // Re c_ij = Re(d^T G_{b_i b_j} d), d = (1, omega)
      const double g00 = Gbb[(2 * i) * 6 + 2 * j].x, g01 = Gbb[(2 * i) * 6 + 2 * j + 1].x;
      const double g10 = Gbb[(2 * i + 1) * 6 + 2 * j].x, g11 = Gbb[(2 * i + 1) * 6 + 2 * j + 1].x;
      const double c = g00 + w * (g01 + g10) + w * w * g11;
      ReX[i * 3 + j] = c + m.lp[i * 3 + j] + m.lp[j * 3 + i];
    }
  double n[3];
  for (int i = 0; i < 3; ++i) {
    // pair index of (i,i) is i
    const double x = ReX[i * 3 + i] + m.qQ[i];
    n[i] = x > 0.0 ? x : 0.0;
  }
  const bool outR = flags & PODP_FLAG_OUT_R;
  for (int e = 0; e < 6; ++e) {
    const int i = kPairI[e], j = kPairJ[e];
    double R = -(a3 / 4.0) * m.qK[e];
    T1[e] = outR ? R : sc[SC_N0 + 3 * i + j] + R;
    I[e] = (w * a3 / 4.0) * (sc[SC_S + 3 * i + j] + nu * m.qM[e] + m.hp[i * 3 + j] + m.hp[j * 3 + i]);
    double mij = 0.0;
    if (i != j) {
      const double x = n[i] + n[j] - 2.0 * (ReX[i * 3 + j] + m.qQ[e]);
      mij = x > 0.0 ? x : 0.0;
    }
    D[e] = a3 / (8.0 * alb) * (n[i] + n[j] + mij);
  }
}

template <int NW>
__global__ void __launch_bounds__(NW * 32) mpt_simple_kernel(EvalArgs a) {
  extern __shared__ double2 smem[];
  const int R = a.L.R;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2 *sP = smem + (size_t)warp * 3 * R;  // P for this warp's omega, [c][i]
  const int64_t total = (int64_t)a.n_obj * a.F;
  for (int64_t t = (int64_t)blockIdx.x * NW + warp; t < total; t += (int64_t)gridDim.x * NW) {
    const int obj = (int)(t / a.F);
    const int64_t f = t - (int64_t)obj * a.F;
    const double *op = a.ops + (size_t)obj * a.L.stride;
    const double w = a.omega[f];
    const double nu = op[a.L.scal + SC_NU];
    const double s = w * nu;
    const double2 *Pw = a.Pws + (size_t)t * 3 * R;
    bool finite = true;
    for (int e = lane; e < 3 * R; e += 32) {
      const double2 v = Pw[e];
      finite &= isfinite(v.x) && isfinite(v.y);
      sP[e] = v;
    }
    finite = __all_sync(0xffffffffu, finite) && isfinite(w);
    __syncwarp();
    double *T1 = a.T1 + (size_t)t * 6, *I = a.I + (size_t)t * 6, *D = a.Delta + (size_t)t * 6;
    if (!finite) {
      const double nan = __longlong_as_double(0x7ff8000000000000ll);
      if (lane < 6) { T1[lane] = nan; I[lane] = nan; D[lane] = nan; }
      continue;
    }
    const double2 *KR = reinterpret_cast<const double2 *>(op + a.L.KR);
    const double2 *Mm = reinterpret_cast<const double2 *>(op + a.L.MI);
    const double2 *Gkk = reinterpret_cast<const double2 *>(op + a.L.Gkk);
    const double2 *Jm = reinterpret_cast<const double2 *>(op + a.L.J);
    const double2 *Gmm = reinterpret_cast<const double2 *>(op + a.L.Gmm);
    const double2 *GbK = reinterpret_cast<const double2 *>(op + a.L.GbK);
    const double2 *GbM = reinterpret_cast<const double2 *>(op + a.L.GbM);
    const double2 *H = reinterpret_cast<const double2 *>(op + a.L.H);
    MptSums m;
#pragma unroll
    for (int e = 0; e < 6; ++e) { m.qK[e] = 0; m.qM[e] = 0; m.qQ[e] = 0; }
#pragma unroll
    for (int e = 0; e < 9; ++e) { m.lp[e] = 0; m.hp[e] = 0; }
    for (int r = lane; r < R; r += 32) {
      double2 yK[3], yM[3], yQ[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) { yK[c] = make_double2(0, 0); yM[c] = yK[c]; yQ[c] = yK[c]; }
      for (int j = 0; j < R; ++j) {
        const double2 kr = __ldg(KR + r * R + j), mm = __ldg(Mm + r * R + j);
        const double2 gk = __ldg(Gkk + r * R + j), jj = __ldg(Jm + r * R + j), gm = __ldg(Gmm + r * R + j);
        // Q = G_KK + s (J + s G_MM)  (Horner)
        const double2 q = make_double2(fma(s, fma(s, gm.x, jj.x), gk.x), fma(s, fma(s, gm.y, jj.y), gk.y));
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double2 p = sP[c * R + j];
          yK[c] = cfma(kr, p, yK[c]);
          yM[c] = cfma(mm, p, yM[c]);
          yQ[c] = cfma(q, p, yQ[c]);
        }
      }
      // Re(conj(p_i[r]) y_j[r]) for the 6 pairs
#pragma unroll
      for (int e = 0; e < 6; ++e) {
        const int i = kPairI[e], j = kPairJ[e];
        const double2 pi = sP[i * R + r];
        m.qK[e] += pi.x * yK[j].x + pi.y * yK[j].y;
        m.qM[e] += pi.x * yM[j].x + pi.y * yM[j].y;
        m.qQ[e] += pi.x * yQ[j].x + pi.y * yQ[j].y;
      }
      // l_i[r] = -(GbK[2i][r] + w GbK[2i+1][r]) - i s (GbM[2i][r] + w GbM[2i+1][r]);  Re(l_i[r] p_j[r]), Re(h_i[r] p_j[r])
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const double2 k0 = GbK[(2 * i) * R + r], k1 = GbK[(2 * i + 1) * R + r];
        const double2 m0 = GbM[(2 * i) * R + r], m1 = GbM[(2 * i + 1) * R + r];
        const double2 gk = make_double2(fma(w, k1.x, k0.x), fma(w, k1.y, k0.y));
        const double2 gm = make_double2(fma(w, m1.x, m0.x), fma(w, m1.y, m0.y));
        const double2 l = make_double2(-gk.x + s * gm.y, -gk.y - s * gm.x);
        const double2 h = H[i * R + r];
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          const double2 pj = sP[j * R + r];
          m.lp[i * 3 + j] += l.x * pj.x - l.y * pj.y;
          m.hp[i * 3 + j] += h.x * pj.x - h.y * pj.y;
        }
      }
    }
#pragma unroll
    for (int e = 0; e < 6; ++e) { m.qK[e] = warp_sum(m.qK[e]); m.qM[e] = warp_sum(m.qM[e]); m.qQ[e] = warp_sum(m.qQ[e]); }
#pragma unroll
    for (int e = 0; e < 9; ++e) { m.lp[e] = warp_sum(m.lp[e]); m.hp[e] = warp_sum(m.hp[e]); }
    if (lane == 0) mpt_epilogue(op, a.L, w, a.flags, m, T1, I, D);
    __syncwarp();
  }
}

cudaError_t launch_mpt(const EvalArgs &a, cudaStream_t s, int *nlaunch) {
  constexpr int NW = 4;
  const int R = a.L.R;
  const size_t sm = (size_t)NW * 3 * R * sizeof(double2);
  const int64_t total = (int64_t)a.n_obj * a.F;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t blocks = (total + NW - 1) / NW;
  if (blocks > (int64_t)sms * 16) blocks = (int64_t)sms * 16;
  mpt_simple_kernel<NW><<<(unsigned)blocks, NW * 32, sm, s>>>(a);
  ++*nlaunch;
  return cudaGetLastError();
}

}  // namespace podp
