// K2 pipelined path: register-resident batched LU with a dedicated pivot warp (rows a2-a3).
//   A(omega) = K + i omega nu M,  B(omega) = b0 + omega b1,  P = A^{-1} B            (eqn:ReducedA)
//
// Roles.  A group works on one frequency at a time with NW "bulk" warps and one "pivot" warp.
//   * Bulk warps hold [A | B] (R x (R+3) complex) in registers, 2-D cyclic: lane = rho + 16*gamma owns rows
//     rho + 16 m and, in bulk warp w, columns w + NW*(gamma + 2 n).  Per elimination step k they only apply the
//     row interchange k <-> p_k, publish U row k and run the rank-1 update with the multipliers L_k.
//   * The pivot warp runs the whole sequential pivot chain, never doing bulk work: it keeps a copy of the next
//     pivot column (lane = row), receives column k as of step k-2 from its owner (who sends it right after
//     updating it in step k-2), applies step k-1 itself (it knows p_{k-1} and L_{k-1}), searches the pivot
//     (redux.sync over an integer magnitude key, lowest row on ties), forms 1/pivot (MUFU.RCP64H + 2 Newton)
//     and the multipliers, publishes them and `bar.arrive`s.  It has the highest warp id on its SMSP, so the
//     hi-warp-id-first issue arbitration gives the critical chain priority over the bulk DFMA streams.
//   Hand-offs: B_k (pivot warp arrives, bulk warps sync) and X_k (column owner arrives, pivot warp syncs), each
//   on two alternating named-barrier ids; multiplier / pivot buffers are 4-deep (the pivot warp may run up to
//   two steps ahead of the slowest bulk warp).
// The bulk steps are fully unrolled (compile-time register indices); the pivot warp is a compact runtime loop.
// B rides along as 3 extra columns; U rows are packed in shared memory; bulk warps 0..2 back-substitute.
#include <cstdlib>
#include <utility>

#include "podp_common.cuh"

namespace podp {

namespace lupw {

__device__ __forceinline__ void bsync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void barrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

template <int R, int NW, int GPB>
struct Cfg {
  static constexpr int NCOL = R + 3;
  static constexpr int MR = (R + 15) / 16;
  static constexpr int CP = 2 * NW;
  static constexpr int NC = (NCOL + CP - 1) / CP;
  static constexpr int LDKM = R + 1;
  static constexpr int NU = R * NCOL - R * (R - 1) / 2;
  static constexpr int NBULK = NW * 32;
  static constexpr int NGRP = (NW + 1) * 32;
  static constexpr int THREADS = GPB * NGRP;
  static constexpr int SM_KM = 2 * R * LDKM;
  static constexpr int SM_GROUP = NU + 4 * R + NCOL + R + 2 * R + 4;  // U, L[4][R], swap, 1/U_kk, colbuf[2][R], ints
  static constexpr size_t BYTES = sizeof(double2) * (size_t)(SM_KM + GPB * SM_GROUP);
  static_assert(R <= 64, "pivot warp holds 2 rows per lane");
  static_assert(GPB * 5 <= 15, "named barrier ids");
};

__host__ __device__ constexpr int uoff(int k, int ncol) { return k * ncol - k * (k - 1) / 2 - k; }

template <int N>
using IC = std::integral_constant<int, N>;

}  // namespace lupw

template <int R, int NW, int GPB>
__global__ void __launch_bounds__(lupw::Cfg<R, NW, GPB>::THREADS, 1) lu_pw_kernel(EvalArgs a) {
  using C = lupw::Cfg<R, NW, GPB>;
  constexpr int NCOL = C::NCOL, MR = C::MR, NC = C::NC, LDKM = C::LDKM, CP = C::CP;
  extern __shared__ double2 smem[];
  double2 *sK = smem, *sM = smem + R * LDKM;
  const int tid = threadIdx.x;
  const int wid = tid >> 5, lane = tid & 31;
  const bool is_pivot = wid >= GPB * NW;
  const int grp = is_pivot ? wid - GPB * NW : wid / NW;
  const int w = is_pivot ? NW : wid % NW;
  const int rho = lane & 15, gam = lane >> 4;
  double2 *sU = smem + C::SM_KM + grp * C::SM_GROUP;
  double2 *sL = sU + C::NU;        // [4][R]
  double2 *sSw = sL + 4 * R;       // [NCOL]
  double2 *sRinv = sSw + NCOL;     // [R]
  double2 *sCol = sRinv + R;       // [2][R]   column hand-off to the pivot warp
  int *sPiv = reinterpret_cast<int *>(sCol + 2 * R);  // [4]
  const int idB = 1 + 5 * grp, idX = idB + 2, idF = idB + 4;
  const int colbase = w + NW * gam;

  const int64_t total = (int64_t)a.n_obj * a.F;
  const int64_t per = (total + gridDim.x - 1) / gridDim.x;
  const int64_t t_begin = (int64_t)blockIdx.x * per;
  const int64_t t_end = t_begin + per < total ? t_begin + per : total;
  const double nanv = __longlong_as_double(0x7ff8000000000000ll);
  const unsigned FULL = 0xffffffffu;

  for (int64_t seg = t_begin; seg < t_end;) {
    const int obj = (int)(seg / a.F);
    const int64_t seg_end_obj = (int64_t)(obj + 1) * a.F;
    const int64_t seg_end = seg_end_obj < t_end ? seg_end_obj : t_end;
    const double *op = a.ops + (size_t)obj * a.L.stride;
    const double nu = op[a.L.scal + SC_NU];
    __syncthreads();
    {
      const double2 *gK = reinterpret_cast<const double2 *>(op + a.L.K);
      const double2 *gM = reinterpret_cast<const double2 *>(op + a.L.M);
      for (int e = tid; e < R * R; e += C::THREADS) {
        const int i = e / R, j = e - i * R;
        sK[i * LDKM + j] = gK[e];
        sM[i * LDKM + j] = gM[e];
      }
    }
    __syncthreads();
    const double2 *gb0 = reinterpret_cast<const double2 *>(op + a.L.b0);
    const double2 *gb1 = reinterpret_cast<const double2 *>(op + a.L.b1);

    for (int64_t t = seg + grp; t < seg_end; t += GPB) {
      const int64_t f = t - (int64_t)obj * a.F;
      const double om = a.omega[f];
      const double s = om * nu;
      const bool om_ok = isfinite(om);

      if (is_pivot) {
        // ================================ pivot warp ================================================================
        // lane owns rows lane and lane + 32 of the current pivot column
        auto column0 = [&](int j, double2 *c) __attribute__((always_inline)) {
#pragma unroll
          for (int m = 0; m < 2; ++m) {
            const int i = lane + 32 * m;
            c[m] = make_double2(0.0, 0.0);
            if (i < R) {
              const double2 k = sK[i * LDKM + j], mm = sM[i * LDKM + j];
              c[m] = make_double2(fma(-s, mm.y, k.x), fma(s, mm.x, k.y));
            }
          }
        };
        double2 lp[2] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
        int pprev = 0;
        bool dead = !om_ok;
        for (int k = 0; k < R; ++k) {
          double2 c[2];
          if (k < 2) {
            column0(k, c);
          } else {
            lupw::bsync(idX + (k & 1), 64);  // column k as of step k-2 is in sCol[k & 1]
#pragma unroll
            for (int m = 0; m < 2; ++m) {
              const int i = lane + 32 * m;
              c[m] = (i < R) ? sCol[(k & 1) * R + i] : make_double2(0.0, 0.0);
            }
          }
          if (!dead) {
            if (k >= 1) {
              // apply step k-1: interchange rows k-1 <-> pprev, then c[i] -= L_{k-1}[i] * u for i > k-1
              const int ra = k - 1, rb = pprev;
              double2 va = ra < 32 ? c[0] : c[1];
              double2 vb = rb < 32 ? c[0] : c[1];
              va.x = __shfl_sync(FULL, va.x, ra & 31);
              va.y = __shfl_sync(FULL, va.y, ra & 31);
              vb.x = __shfl_sync(FULL, vb.x, rb & 31);
              vb.y = __shfl_sync(FULL, vb.y, rb & 31);
              // after the interchange, row ra holds vb (the pivot row's value = u) and row rb holds va
#pragma unroll
              for (int m = 0; m < 2; ++m) {
                const int i = lane + 32 * m;
                if (i == rb && rb != ra) c[m] = va;
                if (i > ra && i < R) c[m] = cfms(lp[m], vb, c[m]);
              }
            }
            // pivot search on column k (rows >= k)
            unsigned key = 0u;
#pragma unroll
            for (int m = 0; m < 2; ++m) {
              const int i = lane + 32 * m;
              const unsigned kk = (mag_key_hi(c[m]) & 0xFFFFFF80u) | (unsigned)(127 - i);
              if (i >= k && i < R && kk > key) key = kk;
            }
            const unsigned best = __reduce_max_sync(FULL, key);
            if ((best >> 7) == 0u) {
              dead = true;
            } else {
              const int p = 127 - (int)(best & 127u);
              double2 pv = p < 32 ? c[0] : c[1];
              double2 dv = k < 32 ? c[0] : c[1];
              pv.x = __shfl_sync(FULL, pv.x, p & 31);
              pv.y = __shfl_sync(FULL, pv.y, p & 31);
              dv.x = __shfl_sync(FULL, dv.x, k & 31);
              dv.y = __shfl_sync(FULL, dv.y, k & 31);
              const double2 rc = crecip_fast(pv);
              double2 *Lout = sL + (k & 3) * R;
#pragma unroll
              for (int m = 0; m < 2; ++m) {
                const int i = lane + 32 * m;
                const bool act = i > k && i < R;
                lp[m] = act ? cmul(i == p ? dv : c[m], rc) : make_double2(0.0, 0.0);
                if (act) Lout[i] = lp[m];
              }
              if (lane == 0) {
                sPiv[k & 3] = p;
                sRinv[k] = rc;
                sU[lupw::uoff(k, NCOL) + k] = pv;
              }
              pprev = p;
            }
          }
          if (dead && lane == 0) sPiv[k & 3] = -1;
          __syncwarp();
          lupw::barrive(idB + (k & 1), C::NGRP);
        }
        lupw::bsync(idF, C::NGRP);   // LU done
        lupw::bsync(idF, C::NGRP);   // back substitution done
        continue;
      }

      // ================================== bulk warps ================================================================
      double2 A[MR][NC];
#pragma unroll
      for (int m = 0; m < MR; ++m) {
        const int i = rho + 16 * m;
#pragma unroll
        for (int n = 0; n < NC; ++n) {
          const int j = colbase + CP * n;
          double2 v = make_double2(0.0, 0.0);
          if (i < R) {
            if (j < R) {
              const double2 k = sK[i * LDKM + j], mm = sM[i * LDKM + j];
              v = make_double2(fma(-s, mm.y, k.x), fma(s, mm.x, k.y));
            } else if (j < NCOL) {
              const double2 x0 = gb0[(j - R) * R + i], x1 = gb1[(j - R) * R + i];
              v = make_double2(fma(om, x1.x, x0.x), fma(om, x1.y, x0.y));
            }
          }
          A[m][n] = v;
        }
      }
      int bad = om_ok ? 0 : -1;

      auto step = [&](auto k_c) __attribute__((always_inline)) {
        constexpr int K = decltype(k_c)::value;
        constexpr int MK = K >> 4, RK = K & 15;
        constexpr bool SEND = K + 2 < R;
        constexpr int K2 = K + 2, W2 = K2 % NW, G2 = (K2 / NW) & 1, N2 = K2 / CP;
        const bool sender = SEND && w == W2;
        lupw::bsync(idB + (K & 1), C::NGRP);
        const int p = sPiv[K & 3];
        if (p < 0 && bad == 0) bad = K + 1;
        if (bad != 0) {
          if constexpr (SEND) {
            if (sender) lupw::barrive(idX + (K2 & 1), 64);
          }
          return;
        }
        const int mp = p >> 4, rp = p & 15;
        double2 *Urow = sU + lupw::uoff(K, NCOL);
        // -- interchange rows K <-> p: publish U row K (= row p), move old row K into row p's slot --------------
        if (p == K) {
#pragma unroll
          for (int n = 0; n < NC; ++n) {
            if (CP * n + CP - 1 > K && CP * n < NCOL) {
              const int j = colbase + CP * n;
              if (rho == RK && j > K && j < NCOL) Urow[j] = A[MK][n];
            }
          }
        } else {
          auto swap_rows = [&](auto m_c) __attribute__((always_inline)) {
            constexpr int M = decltype(m_c)::value;
#pragma unroll
            for (int n = 0; n < NC; ++n) {
              if (CP * n + CP - 1 > K && CP * n < NCOL) {
                const int j = colbase + CP * n;
                const bool act = j > K && j < NCOL;
                if (act && rho == rp) Urow[j] = A[M][n];
                if (act && rho == RK) sSw[j] = A[MK][n];
              }
            }
            __syncwarp();
#pragma unroll
            for (int n = 0; n < NC; ++n) {
              if (CP * n + CP - 1 > K && CP * n < NCOL) {
                const int j = colbase + CP * n;
                if (rho == rp && j > K && j < NCOL) A[M][n] = sSw[j];
              }
            }
          };
          [&]<int... Ms>(std::integer_sequence<int, Ms...>) __attribute__((always_inline)) {
            ((Ms >= MK && mp == Ms ? swap_rows(lupw::IC<Ms>{}) : void()), ...);
          }(std::make_integer_sequence<int, MR>{});
        }
        __syncwarp();
        const double2 *Lin = sL + (K & 3) * R;
        double2 l[MR];
#pragma unroll
        for (int m = 0; m < MR; ++m) {
          l[m] = make_double2(0.0, 0.0);
          if (16 * m + 15 > K && 16 * m < R) {
            const int i = rho + 16 * m;
            if (i > K && i < R) l[m] = Lin[i];
          }
        }
        auto update_slot = [&](auto n_c) __attribute__((always_inline)) {
          constexpr int N = decltype(n_c)::value;
          if constexpr (CP * N + CP - 1 > K && CP * N < NCOL) {
            const int j = colbase + CP * N;
            double2 u = make_double2(0.0, 0.0);
            if (j > K && j < NCOL) u = Urow[j];
#pragma unroll
            for (int m = 0; m < MR; ++m) {
              if (16 * m + 15 > K && 16 * m < R) A[m][N] = cfms(l[m], u, A[m][N]);
            }
          }
        };
        // -- the owner of column K+2 updates it first and hands it to the pivot warp ------------------------------
        if constexpr (SEND) {
          if (sender) {
            update_slot(lupw::IC<N2>{});
            if (gam == G2) {
#pragma unroll
              for (int m = 0; m < MR; ++m) {
                const int i = rho + 16 * m;
                if (i < R) sCol[(K2 & 1) * R + i] = A[m][N2];
              }
            }
            __syncwarp();
            lupw::barrive(idX + (K2 & 1), 64);
          }
        }
        [&]<int... Ns>(std::integer_sequence<int, Ns...>) __attribute__((always_inline)) {
          ((!(SEND && Ns == N2) || !sender ? update_slot(lupw::IC<Ns>{}) : void()), ...);
        }(std::make_integer_sequence<int, NC>{});
      };
      [&]<int... Ks>(std::integer_sequence<int, Ks...>) __attribute__((always_inline)) { (step(lupw::IC<Ks>{}), ...); }(
          std::make_integer_sequence<int, R>{});

      lupw::bsync(idF, C::NGRP);  // LU done (all bulk warps + pivot warp)
      // ---- back substitution U x = y: bulk warp c handles right-hand side c --------------------------------------------
      constexpr int QR = (R + 31) / 32;
      double2 *Pw = a.Pws + (size_t)t * 3 * R;
      for (int c = w; c < 3; c += NW) {
        if (bad == 0) {
          double2 y[QR];
          int ubase[QR];
#pragma unroll
          for (int q = 0; q < QR; ++q) {
            const int i = lane + 32 * q;
            ubase[q] = lupw::uoff(i < R ? i : R - 1, NCOL);
            y[q] = i < R ? sU[ubase[q] + R + c] : make_double2(0.0, 0.0);
          }
          double2 ucol[QR];
#pragma unroll
          for (int q = 0; q < QR; ++q) {
            const int i = lane + 32 * q;
            ucol[q] = (i < R - 1) ? sU[ubase[q] + R - 1] : make_double2(0.0, 0.0);
          }
          double2 rk = sRinv[R - 1];
#pragma unroll
          for (int qb = QR - 1; qb >= 0; --qb) {
            const int khi = (32 * qb + 31 < R - 1) ? 32 * qb + 31 : R - 1;
#pragma unroll 4
            for (int k = khi; k >= 32 * qb; --k) {
              double2 cur[QR];
#pragma unroll
              for (int q = 0; q < QR; ++q) cur[q] = ucol[q];
              const double2 rcur = rk;
              if (k > 0) {
#pragma unroll
                for (int q = 0; q < QR; ++q) {
                  const int i = lane + 32 * q;
                  ucol[q] = (i < k - 1) ? sU[ubase[q] + k - 1] : make_double2(0.0, 0.0);
                }
                rk = sRinv[k - 1];
              }
              double2 yk;
              yk.x = __shfl_sync(FULL, y[qb].x, k & 31);
              yk.y = __shfl_sync(FULL, y[qb].y, k & 31);
              const double2 xk = cmul(yk, rcur);
#pragma unroll
              for (int q = 0; q <= qb; ++q) {
                const int i = lane + 32 * q;
                if (i < k) y[q] = cfms(cur[q], xk, y[q]);
                else if (i == k) y[q] = xk;
              }
            }
          }
#pragma unroll
          for (int q = 0; q < QR; ++q) {
            const int i = lane + 32 * q;
            if (i < R) Pw[c * R + i] = y[q];
            if (a.P_out && i < a.r) reinterpret_cast<double2 *>(a.P_out)[((size_t)t * 3 + c) * a.r + i] = y[q];
          }
        } else {
          for (int i = lane; i < R; i += 32) Pw[c * R + i] = make_double2(nanv, nanv);
          if (a.P_out)
            for (int i = lane; i < a.r; i += 32)
              reinterpret_cast<double2 *>(a.P_out)[((size_t)t * 3 + c) * a.r + i] = make_double2(nanv, nanv);
        }
      }
      if (a.info && w == 0 && lane == 0) a.info[t] = bad;
      lupw::bsync(idF, C::NGRP);  // shared memory free for the next frequency
    }
    seg = seg_end;
  }
}

template <int R, int NW, int GPB>
static cudaError_t launch_lu_pw_t(const EvalArgs &a, cudaStream_t s) {
  using C = lupw::Cfg<R, NW, GPB>;
  auto kern = lu_pw_kernel<R, NW, GPB>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::BYTES);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t total = (int64_t)a.n_obj * a.F;
  int64_t blocks = (total + GPB - 1) / GPB;
  if (blocks > sms) blocks = sms;
  kern<<<(unsigned)blocks, C::THREADS, C::BYTES, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_lu_pw(const EvalArgs &a, cudaStream_t s) {
  if (a.flags & PODP_FLAG_NO_PIVOT) return cudaErrorNotSupported;
  switch (a.L.R) {
    case 48: return launch_lu_pw_t<48, 4, 3>(a, s);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace podp
