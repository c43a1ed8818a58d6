// K2 fast path: register-resident batched shifted complex LU with partial pivoting + 3-RHS solve (rows a2-a3).
//   A(omega) = K + i omega nu M,  B(omega) = b0 + omega b1,  P = A^{-1} B            (eqn:ReducedA)
//
// Layout.  A "group" of NW warps factors one augmented matrix [A | B] (R x (R+3) complex) at a time, held in
// registers.  lane = rho + 16*gamma (rho in [0,16), gamma in [0,2)).  Lane owns rows i = rho + 16 m (m < MR)
// and, in warp w, columns j = w + NW*(gamma + 2 n) (n < NC): 2-D cyclic, so the active trailing block stays
// balanced.  Column k lives in ONE warp (k mod NW), so the pivot search is a single `redux.sync.max` over 32-bit
// keys (fp32 |re|+|im| magnitude bits, row index in the low 7 bits: lowest index wins ties, i.e. LAPACK izamax
// up to the fp32 rounding of the magnitude).  Only the pivot index and the multiplier column cross warps: ONE
// named barrier per elimination step, and the pivot warp of step k+1 updates that column first and searches
// before finishing its step-k update (lookahead).  The row swap and the pivot-row broadcast stay warp-local
// (shared-memory row buffers + __syncwarp); the pivot row's register slot is picked by a warp-uniform branch.
// The elimination loop is fully unrolled: every register index and every retired-slot test is a compile-time
// constant; partially active slots use zero multipliers (an exact no-op).  B rides along as 3 extra columns
// (forward elimination); U rows are stored packed in shared memory and three warps finish with the back
// substitution (one right-hand side each, solution in registers).  K and M are shared-memory resident per CTA.
#include <cstdlib>
#include <utility>

#include "podp_common.cuh"

namespace podp {

namespace lureg {

__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

template <int R, int NW, int GPB>
struct Cfg {
  static constexpr int NCOL = R + 3;
  static constexpr int MR = (R + 15) / 16;
  static constexpr int CP = 2 * NW;                 // column period
  static constexpr int NC = (NCOL + CP - 1) / CP;   // column slots per lane
  static constexpr int LDKM = R + 1;                // padded row stride of K, M in smem
  static constexpr int NU = R * NCOL - R * (R - 1) / 2;  // packed U (row k holds cols k..NCOL-1)
  static constexpr int NT = NW * 32;
  static constexpr int THREADS = NT * GPB;
  static constexpr int SM_KM = 2 * R * LDKM;        // double2
  static constexpr int SM_GROUP = NU + 2 * R + NCOL + R + 2;  // U, L[2][R], swap row, 1/U_kk, ints
  static constexpr size_t BYTES = sizeof(double2) * (size_t)(SM_KM + GPB * SM_GROUP);
  static_assert(R <= 128, "R <= 128");
};

__host__ __device__ constexpr int uoff(int k, int ncol) { return k * ncol - k * (k - 1) / 2 - k; }  // + j

template <int N>
using IC = std::integral_constant<int, N>;

#ifndef PODP_LU_TRACE
#define PODP_LU_TRACE 0
#endif
// dev instrumentation: clock64 stamps of block 0 / group 0 for the first 8 frequencies (compiled out by default)
#define LU_TR(slot)                                                                               \
  do {                                                                                            \
    if constexpr (PODP_LU_TRACE)                                                                  \
      if (a.trace && blockIdx.x == 0 && grp == 0 && lane == 0 && t - seg < 8 * GPB)               \
        a.trace[((t - seg) / GPB) * 1024 + (slot)] = clock64();                                   \
  } while (0)

}  // namespace lureg

template <int R, int NW, int GPB, bool PIV = true>
__global__ void __launch_bounds__(NW * 32 * GPB, 1) lu_reg_kernel(EvalArgs a) {
  using C = lureg::Cfg<R, NW, GPB>;
  constexpr int NCOL = C::NCOL, MR = C::MR, NC = C::NC, LDKM = C::LDKM, CP = C::CP;
  extern __shared__ double2 smem[];
  double2 *sK = smem, *sM = smem + R * LDKM;
  const int tid = threadIdx.x;
  // group g's warps are CTA warps g, g + GPB, g + 2 GPB, ... (with GPB = 4 every group lives on one SMSP)
  const int wid = tid >> 5, lane = tid & 31;
  const int grp = wid % GPB, w = wid / GPB;
  const int gtid = w * 32 + lane;
  const int rho = lane & 15, gam = lane >> 4;
  double2 *sU = smem + C::SM_KM + grp * C::SM_GROUP;
  double2 *sL = sU + C::NU;       // [2][R]
  double2 *sSw = sL + 2 * R;      // [NCOL]
  double2 *sRinv = sSw + NCOL;    // [R]: 1 / U_kk
  int *sPiv = reinterpret_cast<int *>(sRinv + R);  // [2]
  const int bar_id = 1 + 3 * grp;  // ids bar_id, bar_id+1 (alternating steps), bar_id+2 (full group)
  const int colbase = w + NW * gam;  // column of slot n is colbase + CP*n

  const int64_t total = (int64_t)a.n_obj * a.F;
  const int64_t per = (total + gridDim.x - 1) / gridDim.x;
  const int64_t t_begin = (int64_t)blockIdx.x * per;
  const int64_t t_end = t_begin + per < total ? t_begin + per : total;
  const double nanv = __longlong_as_double(0x7ff8000000000000ll);

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
      // ---- a2: assemble my slots of [A | B] ---------------------------------------------------------------
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
      int bad = isfinite(om) ? 0 : -1;  // group-uniform

      // ---- pivot search for step KN (caller guarantees w == KN % NW) -----------------------------------------------
      auto search = [&](auto kn_c) __attribute__((always_inline)) {
        constexpr int KN = decltype(kn_c)::value;
        constexpr int GK = (KN / NW) & 1, NK = KN / CP, MKN = KN >> 4, RKN = KN & 15;
        unsigned best;
        int p;
        if constexpr (PIV) {
          unsigned key = 0u;
#pragma unroll
          for (int m = 0; m < MR; ++m) {
            if (16 * m + 15 >= KN && 16 * m < R) {
              const int i = rho + 16 * m;
              const unsigned kk = (mag_key_hi(A[m][NK]) & 0xFFFFFF80u) | (unsigned)(127 - i);
              const bool cand = gam == GK && i >= KN && i < R;
              key = (cand && kk > key) ? kk : key;
            }
          }
          best = __reduce_max_sync(0xffffffffu, key);
          p = 127 - (int)(best & 127u);
        } else {
          p = KN;
          best = 0xFFFFFFFFu;
        }
        LU_TR(640 + KN);
        const int mp = p >> 4, rp = p & 15;
        double2 pv = A[MKN][NK];
#pragma unroll
        for (int m = MKN + 1; m < MR; ++m)
          if (m == mp) pv = A[m][NK];
        pv.x = __shfl_sync(0xffffffffu, pv.x, rp + 16 * GK);
        pv.y = __shfl_sync(0xffffffffu, pv.y, rp + 16 * GK);
        double2 dv;
        dv.x = __shfl_sync(0xffffffffu, A[MKN][NK].x, RKN + 16 * GK);
        dv.y = __shfl_sync(0xffffffffu, A[MKN][NK].y, RKN + 16 * GK);
        const bool singular = PIV ? (best >> 7) == 0u : (pv.x == 0.0 && pv.y == 0.0);
        LU_TR(768 + KN);
        if (!singular) {
          const double2 rc = crecip_fast(pv);
          LU_TR(832 + KN);
          if (gam == GK) {
            double2 *Lout = sL + (KN & 1) * R;
#pragma unroll
            for (int m = 0; m < MR; ++m) {
              if (16 * m + 15 > KN && 16 * m < R) {
                const int i = rho + 16 * m;
                if (i > KN && i < R) Lout[i] = cmul(i == p ? dv : A[m][NK], rc);
              }
            }
          }
          if (lane == 0) sU[lureg::uoff(KN, NCOL) + KN] = pv;
          if (lane == 1) sRinv[KN] = rc;
        }
        if (lane == 0) sPiv[KN & 1] = singular ? -1 : p;
      };

      // ---- elimination step K: swap rows K <-> p, publish U row K, rank-1 update, lookahead search -------------
      // Barrier protocol: step K's data (pivot p_K, multipliers L_K) is produced by warp K % NW, which
      // `bar.arrive`s on barrier id (K & 1) right after publishing and never waits on it; the other warps
      // `bar.sync` on it.  Alternating ids keep a producer that runs ahead from being counted twice.
      auto step = [&](auto k_c) __attribute__((always_inline)) {
        constexpr int K = decltype(k_c)::value;
        constexpr int MK = K >> 4, RK = K & 15, WK = K % NW;
        LU_TR(K * 4 + w);
        if constexpr (NW > 1) {
          if (w != WK) lureg::named_bar(bar_id + (K & 1), C::NT);
        } else {
          __syncwarp();
        }
        LU_TR(256 + K * 4 + w);
        const int p_raw = sPiv[K & 1];
        if (p_raw < 0 && bad == 0) bad = K + 1;
        const int p = PIV ? p_raw : K;
        constexpr bool HAS_NEXT = K + 1 < R;
        constexpr int K1 = K + 1, W1 = K1 % NW, NK1 = K1 / CP;
        const bool producer = HAS_NEXT && w == W1;
        if (bad != 0) {  // keep the barrier protocol alive: the producer of step K+1 still arrives
          if constexpr (NW > 1 && HAS_NEXT) {
            if (producer) asm volatile("bar.arrive %0, %1;" ::"r"(bar_id + (K1 & 1)), "r"(C::NT) : "memory");
          }
          return;
        }
        const int mp = p >> 4, rp = p & 15;
        double2 *Urow = sU + lureg::uoff(K, NCOL);
        // multipliers of my active rows
        const double2 *Lin = sL + (K & 1) * R;
        double2 l[MR];
#pragma unroll
        for (int m = 0; m < MR; ++m) {
          l[m] = make_double2(0.0, 0.0);
          if (16 * m + 15 > K && 16 * m < R) {
            const int i = rho + 16 * m;
            if (i > K && i < R) l[m] = Lin[i];
          }
        }
        // -- lookahead (producer of step K+1): swap + update column slot NK1 through shuffles, then search --------
        if constexpr (HAS_NEXT) {
          if (producer) {
            const int j = colbase + CP * NK1;
            const bool valid = j > K && j < NCOL;
            double2 pr = A[MK][NK1];  // will hold the pivot row's value (row p) of my column
            double2 ok = A[MK][NK1];  // old row K value of my column
#pragma unroll
            for (int m = MK + 1; m < MR; ++m)
              if (m == mp) pr = A[m][NK1];
            const int half = 16 * gam;
            double2 u, rowk;
            u.x = __shfl_sync(0xffffffffu, pr.x, rp + half);
            u.y = __shfl_sync(0xffffffffu, pr.y, rp + half);
            rowk.x = __shfl_sync(0xffffffffu, ok.x, RK + half);
            rowk.y = __shfl_sync(0xffffffffu, ok.y, RK + half);
            if (rho == rp && valid) Urow[j] = u;
            if (!valid) u = make_double2(0.0, 0.0);
#pragma unroll
            for (int m = 0; m < MR; ++m) {
              if (16 * m + 15 > K && 16 * m < R) {
                double2 x = A[m][NK1];
                if (p != K && rho == rp && m == mp && valid) x = rowk;
                A[m][NK1] = cfms(l[m], u, x);
              }
            }
            LU_TR(512 + K);
            search(lureg::IC<K1>{});
            LU_TR(576 + K);
            if constexpr (NW > 1) asm volatile("bar.arrive %0, %1;" ::"r"(bar_id + (K1 & 1)), "r"(C::NT) : "memory");
          }
        }
        // -- publish U row K (= current row p) / stash old row K, then receive (all slots but the lookahead one) ---
        auto skip = [&](int n) __attribute__((always_inline)) { return HAS_NEXT && producer && n == NK1; };
        if (p == K) {
#pragma unroll
          for (int n = 0; n < NC; ++n) {
            if (CP * n + CP - 1 > K && CP * n < NCOL) {
              const int j = colbase + CP * n;
              if (!skip(n) && rho == RK && j > K && j < NCOL) Urow[j] = A[MK][n];
            }
          }
        } else {
          auto swap_rows = [&](auto m_c) __attribute__((always_inline)) {
            constexpr int M = decltype(m_c)::value;
#pragma unroll
            for (int n = 0; n < NC; ++n) {
              if (CP * n + CP - 1 > K && CP * n < NCOL) {
                const int j = colbase + CP * n;
                const bool act = !skip(n) && j > K && j < NCOL;
                if (act && rho == rp) Urow[j] = A[M][n];
                if (act && rho == RK) sSw[j] = A[MK][n];
              }
            }
            __syncwarp();
#pragma unroll
            for (int n = 0; n < NC; ++n) {
              if (CP * n + CP - 1 > K && CP * n < NCOL) {
                const int j = colbase + CP * n;
                if (!skip(n) && rho == rp && j > K && j < NCOL) A[M][n] = sSw[j];
              }
            }
          };
          [&]<int... Ms>(std::integer_sequence<int, Ms...>) __attribute__((always_inline)) {
            ((Ms >= MK && mp == Ms ? swap_rows(lureg::IC<Ms>{}) : void()), ...);
          }(std::make_integer_sequence<int, MR>{});
        }
        __syncwarp();
        // -- rank-1 update of the remaining slots -------------------------------------------------------------------
        auto update_slot = [&](auto n_c) __attribute__((always_inline)) {
          constexpr int N = decltype(n_c)::value;
          if constexpr (CP * N + CP - 1 > K && CP * N < NCOL) {
            if (skip(N)) return;
            const int j = colbase + CP * N;
            double2 u = make_double2(0.0, 0.0);
            if (j > K && j < NCOL) u = Urow[j];
#pragma unroll
            for (int m = 0; m < MR; ++m) {
              if (16 * m + 15 > K && 16 * m < R) A[m][N] = cfms(l[m], u, A[m][N]);
            }
          }
        };
        [&]<int... Ns>(std::integer_sequence<int, Ns...>) __attribute__((always_inline)) { (update_slot(lureg::IC<Ns>{}), ...); }(
            std::make_integer_sequence<int, NC>{});
      };

      if (w == 0) {
        if (bad == 0) search(lureg::IC<0>{});
        else if (lane == 0) sPiv[0] = -1;
        __syncwarp();
        if constexpr (NW > 1) asm volatile("bar.arrive %0, %1;" ::"r"(bar_id), "r"(C::NT) : "memory");
      }
      [&]<int... Ks>(std::integer_sequence<int, Ks...>) __attribute__((always_inline)) { (step(lureg::IC<Ks>{}), ...); }(
          std::make_integer_sequence<int, R>{});

      if constexpr (NW > 1) lureg::named_bar(bar_id + 2, C::NT); else __syncwarp();
      LU_TR(700 + w);
      // ---- back substitution U x = y: warp c handles right-hand side c (y in registers, U from smem) ----------
      //      chain per k: shfl y_k -> x_k = y_k / U_kk -> y_{k-1} -= U_{k-1,k} x_k; U column k+... prefetched.
      constexpr int QR = (R + 31) / 32;
      double2 *Pw = a.Pws + (size_t)t * 3 * R;
      for (int c = w; c < 3; c += NW) {
        if (bad == 0) {
          double2 y[QR];
          int ubase[QR];
#pragma unroll
          for (int q = 0; q < QR; ++q) {
            const int i = lane + 32 * q;
            ubase[q] = lureg::uoff(i < R ? i : R - 1, NCOL);
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
              if (k > 0) {  // prefetch column k-1 of U (rows above it) and 1/U_{k-1,k-1}
#pragma unroll
                for (int q = 0; q < QR; ++q) {
                  const int i = lane + 32 * q;
                  ucol[q] = (i < k - 1) ? sU[ubase[q] + k - 1] : make_double2(0.0, 0.0);
                }
                rk = sRinv[k - 1];
              }
              double2 yk;
              yk.x = __shfl_sync(0xffffffffu, y[qb].x, k & 31);
              yk.y = __shfl_sync(0xffffffffu, y[qb].y, k & 31);
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
      LU_TR(708 + w);
      if (a.info && gtid == 0) a.info[t] = bad;
      if constexpr (NW > 1) lureg::named_bar(bar_id + 2, C::NT); else __syncwarp();
    }
    seg = seg_end;
  }
}

template <int R, int NW, int GPB, bool PIV = true>
static cudaError_t launch_lu_reg_t(const EvalArgs &a, cudaStream_t s) {
  using C = lureg::Cfg<R, NW, GPB>;
  auto kern = lu_reg_kernel<R, NW, GPB, PIV>;
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

// Returns cudaErrorNotSupported when no register-resident instantiation exists for this R / flags.
cudaError_t launch_lu_reg(const EvalArgs &a, cudaStream_t s) {
  if (a.flags & PODP_FLAG_NO_PIVOT) {
    if (a.L.R == 48) return launch_lu_reg_t<48, 4, 4, false>(a, s);
    return cudaErrorNotSupported;
  }
  switch (a.L.R) {
    case 48:
      return launch_lu_reg_t<48, 4, 4>(a, s);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace podp
