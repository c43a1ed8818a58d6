// K3 alternative for the A/B of north_star's design (PODP_FLAG_MPT_GEMM): the MPT quadratic forms and the
// certificate's Q(omega) forms as FP64 tensor-core GEMMs over the solution panel, operands staged by the bulk-copy
// (TMA) engine.  Same quantities as mpt_tile_kernel (rows a4-a6: eqn:podprealmpt P:600-604, eqn:podpimagmpt
// P:606-620, lemma:certificate P:632-661 in the form X_ij = c_ij + l_i p_j + conj(l_j p_i) + p_i^H Q p_j).
//
// A CTA takes NF = 16 consecutive frequencies of one object: their P (R x 48 complex: column n = 3 f + i) is
// bulk-copied (cp.async.bulk, one 16R-byte column per copy, SASS UBLKCP) into shared memory with a padded row so the
// B fragments are bank-conflict free.  The units (operator o in {K_R, M_I, G_KK, J, G_MM}) x (8-row block of the
// operator) are spread over the 8 warps; a unit's 8 operator rows are bulk-copied into a per-warp double buffer
// (mbarrier completion) while the previous unit computes Y = X P on mma.sync.m8n8k4.f64 (a complex 8x8x4 step =
// 4 DMMA per column group of 8), and the unit then contracts its 8 rows of Y with conj(P) into the 9 (i, j) sums per
// frequency (shuffle reduction over the rows, shared-memory atomics over the row blocks).  Q(omega) = G_KK + s J +
// s^2 G_MM is combined after the GEMMs (so 120 r^2 flops per frequency execute against F_alg's 80 r^2: the Horner
// formation of Q per frequency has no GEMM form).  The linear terms and the epilogue run one warp per frequency.
#include "podp_common.cuh"

namespace podp {

namespace mptg {

constexpr int NF = 16;       // frequencies per CTA tile
constexpr int NC = 3 * NF;   // complex columns of the P tile
constexpr int NG = NC / 8;   // column groups of 8 (DMMA n)
constexpr int WARPS = 8;

template <int R>
struct Cfg {
  static constexpr int LDP = R + 1;                        // padded column stride of the P tile (complex)
  static constexpr int P_BYTES = NC * LDP * 16;
  static constexpr int XBUF = 8 * R * 16;                  // one unit's 8 operator rows
  static constexpr int Q_BYTES = 5 * NF * 9 * 8;
  // operator-row buffers per warp: double-buffered where shared memory allows (not at R = 96)
  static constexpr int NBUF = P_BYTES + WARPS * 2 * XBUF + Q_BYTES + 256 <= 227 * 1024 ? 2 : 1;
  static constexpr int BYTES = P_BYTES + WARPS * NBUF * XBUF + Q_BYTES + 64 + WARPS * 2 * 8;
  static constexpr int UNITS = 5 * (R / 8);
};

__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *m, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *m, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *m, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(m)), "r"(parity)
        : "memory");
  }
}
// bulk copy global -> shared (the TMA engine's 1-D mode), completion counted on mbarrier m
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *m) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(m))
               : "memory");
}

}  // namespace mptg

template <int R>
__global__ void __launch_bounds__(mptg::WARPS * 32, 1) mpt_gemm_kernel(EvalArgs a) {
  using C = mptg::Cfg<R>;
  using namespace mptg;
  constexpr int LDP = C::LDP, NRB = R / 8;
  extern __shared__ __align__(128) unsigned char smem[];
  double2 *sP = reinterpret_cast<double2 *>(smem);
  constexpr int NB = C::NBUF;
  double2 *sX = reinterpret_cast<double2 *>(smem + C::P_BYTES);  // [warp][NBUF][8 R]
  double *sQ = reinterpret_cast<double *>(smem + C::P_BYTES + WARPS * NB * C::XBUF);  // [o][f][9]
  uint64_t *mbP = reinterpret_cast<uint64_t *>(smem + C::P_BYTES + WARPS * NB * C::XBUF + C::Q_BYTES);
  uint64_t *mbX = mbP + 8;  // [warp][2]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, r4 = lane >> 2, q = lane & 3;
  const double *op = a.ops;  // one object (the launcher enforces n_obj == 1)
  const int64_t ntiles = (a.F + NF - 1) / NF;
  if (threadIdx.x == 0) {
    mbar_init(mbP, 1);
    for (int i = 0; i < 2 * WARPS; ++i) mbar_init(mbX + i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t parP = 0, parX[2] = {0, 0};
  const double2 *ops5[5] = {reinterpret_cast<const double2 *>(op + a.L.KR), reinterpret_cast<const double2 *>(op + a.L.MI),
                            reinterpret_cast<const double2 *>(op + a.L.Gkk), reinterpret_cast<const double2 *>(op + a.L.J),
                            reinterpret_cast<const double2 *>(op + a.L.Gmm)};
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t f0 = tile * NF;
    const int nf = (int)(a.F - f0 < NF ? a.F - f0 : NF);
    // ---- the P tile: one bulk copy per (frequency, direction) column; absent frequencies' columns zeroed ----------
    if (threadIdx.x == 0) {
      mbar_expect_tx(mbP, (uint32_t)(3 * nf * R * 16));
      for (int n = 0; n < 3 * nf; ++n)
        mptg::bulk_g2s(sP + n * LDP, a.Pws + ((size_t)(f0 + n / 3) * 3 + n % 3) * R, R * 16, mbP);
    }
    for (int e = threadIdx.x; e < 5 * NF * 9; e += blockDim.x) sQ[e] = 0.0;
    for (int e = threadIdx.x; e < (NC - 3 * nf) * LDP; e += blockDim.x) sP[3 * nf * LDP + e] = make_double2(0.0, 0.0);
    // ---- units (operator, 8-row block), double-buffered bulk copies of the operator rows ------------------------
    int slot = 0;
    auto issue = [&](int u, int buf) {
      if (lane == 0) {
        const int o = u / NRB, rb = u % NRB;
        mbar_expect_tx(mbX + 2 * warp + buf, (uint32_t)(8 * R * 16));
        mptg::bulk_g2s(sX + (size_t)(NB * warp + buf) * 8 * R, ops5[o] + (size_t)rb * 8 * R, 8 * R * 16,
                       mbX + 2 * warp + buf);
      }
    };
    if (warp < C::UNITS) issue(warp, 0);
    mbar_wait(mbP, parP);
    parP ^= 1u;
    __syncthreads();  // P tile complete and zero-filled, sQ zeroed
    for (int u = warp; u < C::UNITS; u += WARPS, slot ^= (NB - 1)) {
      if (NB == 2 && u + WARPS < C::UNITS) issue(u + WARPS, slot ^ 1);
      mbar_wait(mbX + 2 * warp + slot, parX[slot]);
      parX[slot] ^= 1u;
      const double2 *X = sX + (size_t)(NB * warp + slot) * 8 * R;  // rows 8 rb .. 8 rb + 7, row-major
      double cr[NG][2], ci[NG][2];
#pragma unroll
      for (int g = 0; g < NG; ++g) cr[g][0] = cr[g][1] = ci[g][0] = ci[g][1] = 0.0;
#pragma unroll 4
      for (int k0 = 0; k0 < R; k0 += 4) {
        const double2 x = X[r4 * R + k0 + q];  // A fragment: row r4, k = k0 + q
#pragma unroll
        for (int g = 0; g < NG; ++g) {
          const double2 p = sP[(8 * g + r4) * LDP + k0 + q];  // B fragment: k = k0 + q, n = 8 g + r4
          dmma(cr[g][0], cr[g][1], x.x, p.x);
          dmma(cr[g][0], cr[g][1], -x.y, p.y);
          dmma(ci[g][0], ci[g][1], x.x, p.y);
          dmma(ci[g][0], ci[g][1], x.y, p.x);
        }
      }
      __syncwarp();  // X buffer free for the next copy into it
      if (NB == 1 && u + WARPS < C::UNITS) issue(u + WARPS, 0);
      // contraction: sum over this unit's rows a of Re(conj(P[a, (f, i)]) Y[a, (f, j)]), Y in C fragments
      const int o = u / NRB, a0 = (u % NRB) * 8 + r4;
      double part[NG][2][3];
#pragma unroll
      for (int g = 0; g < NG; ++g)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int n = 8 * g + 2 * q + e, f = n / 3;
#pragma unroll
          for (int i = 0; i < 3; ++i) {
            const double2 pa = sP[(3 * f + i) * LDP + a0];
            part[g][e][i] = fma(pa.x, e ? cr[g][1] : cr[g][0], pa.y * (e ? ci[g][1] : ci[g][0]));
          }
        }
#pragma unroll
      for (int g = 0; g < NG; ++g)
#pragma unroll
        for (int e = 0; e < 2; ++e)
#pragma unroll
          for (int i = 0; i < 3; ++i) {
            double v = part[g][e][i];
            v += __shfl_xor_sync(0xffffffffu, v, 4);
            v += __shfl_xor_sync(0xffffffffu, v, 8);
            v += __shfl_xor_sync(0xffffffffu, v, 16);
            part[g][e][i] = v;
          }
      if (r4 == 0) {
#pragma unroll
        for (int g = 0; g < NG; ++g)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int n = 8 * g + 2 * q + e, f = n / 3, j = n % 3;
#pragma unroll
            for (int i = 0; i < 3; ++i) atomicAdd(sQ + (o * NF + f) * 9 + i * 3 + j, part[g][e][i]);
          }
      }
    }
    __syncthreads();
    // ---- linear terms and epilogue: warp w handles frequencies w and w + 8 -------------------------------------
    for (int fl = warp; fl < nf; fl += WARPS) {
      const int64_t f = f0 + fl;
      const double w = a.omega[f];
      const double nu = op[a.L.scal + SC_NU];
      const double s = w * nu;
      const double2 *GbK = reinterpret_cast<const double2 *>(op + a.L.GbK);
      const double2 *GbM = reinterpret_cast<const double2 *>(op + a.L.GbM);
      const double2 *H = reinterpret_cast<const double2 *>(op + a.L.H);
      double lp[9], hp[9];
#pragma unroll
      for (int e = 0; e < 9; ++e) lp[e] = hp[e] = 0.0;
      for (int b = lane; b < R; b += 32) {
        double2 p[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) p[c] = sP[(3 * fl + c) * LDP + b];
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
            lp[i * 3 + j] = fma(l.x, p[j].x, fma(-l.y, p[j].y, lp[i * 3 + j]));
            hp[i * 3 + j] = fma(h.x, p[j].x, fma(-h.y, p[j].y, hp[i * 3 + j]));
          }
        }
      }
#pragma unroll
      for (int o2 = 16; o2; o2 >>= 1)
#pragma unroll
        for (int e = 0; e < 9; ++e) {
          lp[e] += __shfl_xor_sync(0xffffffffu, lp[e], o2);
          hp[e] += __shfl_xor_sync(0xffffffffu, hp[e], o2);
        }
      if (lane == 0) {
        const double *sq = sQ + fl * 9;  // operator o at sq + o NF 9
        double qK[6], qM[6], qQ[6];
        bool ok = isfinite(w);
#pragma unroll
        for (int e = 0; e < 6; ++e) {
          const int i = e < 3 ? e : (e < 5 ? 0 : 1);
          const int j = e < 3 ? e : (e == 3 ? 1 : 2);
          qK[e] = sq[0 * NF * 9 + i * 3 + j];
          qM[e] = sq[1 * NF * 9 + i * 3 + j];
          qQ[e] = fma(s, fma(s, sq[4 * NF * 9 + i * 3 + j], sq[3 * NF * 9 + i * 3 + j]), sq[2 * NF * 9 + i * 3 + j]);
          ok &= isfinite(qK[e]) && isfinite(qM[e]) && isfinite(qQ[e]);
        }
#pragma unroll
        for (int e = 0; e < 9; ++e) ok &= isfinite(lp[e]) && isfinite(hp[e]);
        double *T1p = a.T1 + (size_t)f * 6, *Ip = a.I + (size_t)f * 6, *Dp = a.Delta + (size_t)f * 6;
        const double nanv = __longlong_as_double(0x7ff8000000000000ll);
        if (!ok) {
          for (int e = 0; e < 6; ++e) T1p[e] = Ip[e] = Dp[e] = nanv;
        } else {
          const double *sc = op + a.L.scal;
          const double alpha = sc[SC_ALPHA], alb = sc[SC_ALPHA_LB];
          const double a3 = alpha * alpha * alpha;
          const double2 *Gbb = reinterpret_cast<const double2 *>(op + a.L.Gbb);
          double ReX[9];
          for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) {
              const double g00 = Gbb[(2 * i) * 6 + 2 * j].x, g01 = Gbb[(2 * i) * 6 + 2 * j + 1].x;
              const double g10 = Gbb[(2 * i + 1) * 6 + 2 * j].x, g11 = Gbb[(2 * i + 1) * 6 + 2 * j + 1].x;
              const double c = g00 + w * (g01 + g10) + w * w * g11;
              ReX[i * 3 + j] = c + lp[i * 3 + j] + lp[j * 3 + i];
            }
          double n3[3];
          for (int i = 0; i < 3; ++i) {
            const double x = ReX[i * 3 + i] + qQ[i];
            n3[i] = x > 0.0 ? x : 0.0;
          }
          const bool outR = a.flags & PODP_FLAG_OUT_R;
          for (int e = 0; e < 6; ++e) {
            const int i = e < 3 ? e : (e < 5 ? 0 : 1);
            const int j = e < 3 ? e : (e == 3 ? 1 : 2);
            const double Rv = -(a3 / 4.0) * qK[e];
            T1p[e] = outR ? Rv : sc[SC_N0 + 3 * i + j] + Rv;
            Ip[e] = (w * a3 / 4.0) * (sc[SC_S + 3 * i + j] + nu * qM[e] + hp[i * 3 + j] + hp[j * 3 + i]);
            double mij = 0.0;
            if (i != j) {
              const double x = n3[i] + n3[j] - 2.0 * (ReX[i * 3 + j] + qQ[e]);
              mij = x > 0.0 ? x : 0.0;
            }
            Dp[e] = a3 / (8.0 * alb) * (n3[i] + n3[j] + mij);
          }
        }
      }
    }
    __syncthreads();  // sP and sQ are rewritten by the next tile
  }
}

template <int R>
static cudaError_t launch_mpt_gemm_t(const EvalArgs &a, cudaStream_t s, int sms) {
  using C = mptg::Cfg<R>;
  auto kern = mpt_gemm_kernel<R>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::BYTES);
  if (e != cudaSuccess) return e;
  const int64_t tiles = (a.F + mptg::NF - 1) / mptg::NF;
  const int64_t blocks = tiles < sms ? tiles : sms;
  kern<<<(unsigned)blocks, mptg::WARPS * 32, C::BYTES, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_mpt_gemm(const EvalArgs &a, cudaStream_t s, int sms) {
  if (a.n_obj != 1) return cudaErrorNotSupported;
  switch (a.L.R) {
    case 24: return launch_mpt_gemm_t<24>(a, s, sms);
    case 48: return launch_mpt_gemm_t<48>(a, s, sms);
    case 96: return launch_mpt_gemm_t<96>(a, s, sms);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace podp
