// K2 blocked path: one warp per frequency, panel-blocked right-looking LU with partial pivoting + 3-RHS solve
// (rows a2-a3).   A(omega) = K + i omega nu M,  B(omega) = b0 + omega b1,  P = A^{-1} B   (eqn:ReducedA)
//
// Layout / algorithm (per warp, no inter-warp synchronisation at all):
//   * [A | B] (R x (R+3) complex, zero-padded to R x NCP) lives in the warp's slice of shared memory.
//   * For each panel of NB = 8 columns: the panel rows kb..R-1 are held in registers (lane = row, MS slots) and
//     factored with partial pivoting (redux.sync argmax of an integer magnitude key, lowest row on ties; row swap
//     by shuffles; pivot reciprocal by MUFU.RCP64H + 2 Newton steps); the 8 row interchanges are then applied to
//     the columns right of the panel, U12 = L11^{-1} A12 is formed column-wise, and the trailing block
//     A22 -= L21 U12 runs on the FP64 tensor path (mma.sync.m8n8k4.f64 -> DMMA.8x8x4; a complex 8x8x4 product
//     is 4 real DMMAs) over 8x8 complex tiles whose C fragments are read/written in shared memory.
//   * The 3 right-hand sides ride along as columns R..R+2 (forward elimination); back substitution runs from the
//     U rows in shared memory with the solution column in registers.
#include <cstdlib>

#include "podp_common.cuh"

namespace podp {

namespace lublk {

constexpr int NB = 8;

template <int R>
struct Cfg {
  static_assert(R % 8 == 0, "R must be a multiple of 8 (exact padding)");
  static constexpr int NCP = R + 8;             // columns incl. RHS block (R..R+2) padded to a tile
  static constexpr int LDA = NCP + 4;           // row stride (complex): LDA = 4 mod 8 for conflict-light tiles
  static constexpr int MS = (R + 31) / 32;      // panel row slots per lane
  static constexpr int A_ELEMS = R * LDA;
  static constexpr int W_BYTES = A_ELEMS * 16 + R * 16 + 2 * 8 * 16 + R * 4 + 16;  // A, 1/U_kk, 2 scratch rows, pivots
  static constexpr int WARPS = (200 * 1024) / W_BYTES > 16 ? 16 : (200 * 1024) / W_BYTES;
  static constexpr size_t BYTES = (size_t)WARPS * W_BYTES;
};

__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

#ifndef PODP_LU_TRACE
#define PODP_LU_TRACE 0
#endif
}  // namespace lublk
// dev instrumentation: clock64 stamps of block 0 / warp 0 for its first 4 frequencies (compiled out by default)
#define LB_TR(slot)                                                                                \
  do {                                                                                             \
    if constexpr (PODP_LU_TRACE)                                                                   \
      if (a.trace && blockIdx.x == 0 && warp == 0 && lane == 0 && it_ < 4)                        \
        a.trace[it_ * 1024 + (slot)] = clock64();                                                 \
  } while (0)

template <int R>
__global__ void __launch_bounds__(lublk::Cfg<R>::WARPS * 32, 1) lu_blk_kernel(EvalArgs a) {
  using C = lublk::Cfg<R>;
  constexpr int NCP = C::NCP, LDA = C::LDA, MS = C::MS, NB = lublk::NB, NCOL = R + 3;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char *wbase = smem_raw + (size_t)warp * C::W_BYTES;
  double2 *A = reinterpret_cast<double2 *>(wbase);
  double2 *sRinv = A + C::A_ELEMS;
  double2 *sRowK = sRinv + R, *sRowP = sRowK + NB;  // panel row scratch (old row k, pivot row)
  int *sPiv = reinterpret_cast<int *>(sRowP + NB);
  const int64_t total = (int64_t)a.n_obj * a.F;
  const double nanv = __longlong_as_double(0x7ff8000000000000ll);
  const unsigned FULL = 0xffffffffu;

  int it_ = -1;
  for (int64_t t = (int64_t)blockIdx.x * C::WARPS + warp; t < total; t += (int64_t)gridDim.x * C::WARPS) {
    ++it_;
    const int obj = (int)(t / a.F);
    const int64_t f = t - (int64_t)obj * a.F;
    const double *op = a.ops + (size_t)obj * a.L.stride;
    const double om = a.omega[f];
    const double s = om * op[a.L.scal + SC_NU];
    LB_TR(0);
    // ---- a2: assemble [A | B | 0] ----------------------------------------------------------------------------
    {
      const double2 *gK = reinterpret_cast<const double2 *>(op + a.L.K);
      const double2 *gM = reinterpret_cast<const double2 *>(op + a.L.M);
      static_assert((R * R) % 32 == 0, "R*R must be a multiple of 32");
      constexpr int PER = (R * R) / 32;
      constexpr int BATCH = 12;
#pragma unroll 1
      for (int e0 = 0; e0 < PER; e0 += BATCH) {
        double2 kk[BATCH], mm[BATCH];
#pragma unroll
        for (int q = 0; q < BATCH; ++q) {
          const int e = (e0 + q) * 32 + lane;
          if (e0 + q < PER) {
            kk[q] = __ldg(gK + e);
            mm[q] = __ldg(gM + e);
          }
        }
#pragma unroll
        for (int q = 0; q < BATCH; ++q) {
          const int e = (e0 + q) * 32 + lane;
          if (e0 + q < PER) {
            const int i = e / R, j = e - i * R;
            A[i * LDA + j] = make_double2(fma(-s, mm[q].y, kk[q].x), fma(s, mm[q].x, kk[q].y));
          }
        }
      }
      const double2 *gb0 = reinterpret_cast<const double2 *>(op + a.L.b0);
      const double2 *gb1 = reinterpret_cast<const double2 *>(op + a.L.b1);
      for (int e = lane; e < 8 * R; e += 32) {
        const int i = e >> 3, c = e & 7;
        double2 v = make_double2(0.0, 0.0);
        if (c < 3) {
          const double2 x0 = __ldg(gb0 + c * R + i), x1 = __ldg(gb1 + c * R + i);
          v = make_double2(fma(om, x1.x, x0.x), fma(om, x1.y, x0.y));
        }
        A[i * LDA + R + c] = v;
      }
    }
    __syncwarp();
    LB_TR(1);
    int info = isfinite(om) ? 0 : -1;

    // ---- a3: blocked LU with partial pivoting --------------------------------------------------------------------
    for (int kb = 0; kb < R && info == 0; kb += NB) {
      LB_TR(16 + (kb / NB) * 4);
      // (1) panel factorisation in registers: lane owns rows kb + lane + 32 m
      double2 pn[MS][NB];
#pragma unroll
      for (int m = 0; m < MS; ++m) {
        const int i = kb + lane + 32 * m;
#pragma unroll
        for (int c = 0; c < NB; ++c) pn[m][c] = (i < R) ? A[i * LDA + kb + c] : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        const int kr = kb + j;  // pivot row position (held by lane j, slot 0)
        unsigned key = 0u;
#pragma unroll
        for (int m = 0; m < MS; ++m) {
          const int i = kb + lane + 32 * m;
          const unsigned kk = (mag_key_hi(pn[m][j]) & 0xFFFFFF80u) | (unsigned)(127 - i);
          if (i >= kr && i < R && kk > key) key = kk;
        }
        const unsigned best = __reduce_max_sync(FULL, key);
        if ((best >> 7) == 0u) {  // exactly zero pivot column
          info = kr + 1;
          break;
        }
        const int p = 127 - (int)(best & 127u);
        const int lp = (p - kb) & 31, mp = (p - kb) >> 5;
        if (lane == 0) sPiv[kr] = p;
        // stage row kr (lane j, slot 0) and the pivot row p (lane lp, slot mp) in shared memory
        if (lane == j) {
#pragma unroll
          for (int c = 0; c < NB; ++c) sRowK[c] = pn[0][c];
        }
        if (lane == lp) {
#pragma unroll
          for (int m = 0; m < MS; ++m)
            if (m == mp) {
#pragma unroll
              for (int c = 0; c < NB; ++c) sRowP[c] = pn[m][c];
            }
        }
        __syncwarp();
        if (p != kr) {
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
        const double2 pv = sRowP[j];
        const double2 rc = crecip_fast(pv);
        if (lane == 0) sRinv[kr] = rc;
        double2 l[MS];
#pragma unroll
        for (int m = 0; m < MS; ++m) {
          const int i = kb + lane + 32 * m;
          l[m] = (i > kr && i < R) ? cmul(pn[m][j], rc) : make_double2(0.0, 0.0);
          if (i > kr && i < R) pn[m][j] = l[m];
        }
#pragma unroll
        for (int c = j + 1; c < NB; ++c) {
          const double2 u = sRowP[c];
#pragma unroll
          for (int m = 0; m < MS; ++m) pn[m][c] = cfms(l[m], u, pn[m][c]);
        }
        __syncwarp();  // scratch rows reused by the next column
      }
      if (info != 0) break;
      // write the factored panel back (L21 multipliers, U11)
#pragma unroll
      for (int m = 0; m < MS; ++m) {
        const int i = kb + lane + 32 * m;
        if (i < R) {
#pragma unroll
          for (int c = 0; c < NB; ++c) A[i * LDA + kb + c] = pn[m][c];
        }
      }
      __syncwarp();
      LB_TR(17 + (kb / NB) * 4);
      // (2) row interchanges + U12 = L11^{-1} A12 for the columns right of the panel (lane = column)
      for (int col = kb + NB + lane; col < NCP; col += 32) {
        double2 x[NB];
#pragma unroll
        for (int j = 0; j < NB; ++j) {
          const int p = sPiv[kb + j];
          const double2 vk = A[(kb + j) * LDA + col];
          if (p != kb + j) {
            const double2 vp = A[p * LDA + col];
            A[p * LDA + col] = vk;
            x[j] = vp;
          } else {
            x[j] = vk;
          }
          // rows kb+j' (j' > j) not yet swapped may be read later: keep swapped values in registers only
          A[(kb + j) * LDA + col] = x[j];
        }
#pragma unroll
        for (int j = 1; j < NB; ++j) {
#pragma unroll
          for (int tt = 0; tt < j; ++tt) x[j] = cfms(A[(kb + j) * LDA + kb + tt], x[tt], x[j]);
        }
#pragma unroll
        for (int j = 0; j < NB; ++j) A[(kb + j) * LDA + col] = x[j];
      }
      __syncwarp();
      LB_TR(18 + (kb / NB) * 4);
      // (3) trailing update A22 -= L21 U12 on 8x8 complex tiles (DMMA)
      const int r0 = kb + NB;
      const int arow = lane >> 2, acol = lane & 3;   // A fragment (8x4): row, k
      const int bk = lane & 3, bcol = lane >> 2;      // B fragment (4x8): k, col
      const int crow = lane >> 2, ccol = 2 * (lane & 3);
      for (int tr = r0; tr < R; tr += 8) {
        // A fragments (L21 rows tr..tr+7, k = kb..kb+7): two k-steps of 4
        const double2 a0 = A[(tr + arow) * LDA + kb + acol];
        const double2 a1 = A[(tr + arow) * LDA + kb + 4 + acol];
        auto tile = [&](double &cr0, double &cr1, double &ci0, double &ci1, double2 b0, double2 b1)
            __attribute__((always_inline)) {
          // C -= A B  (complex): C_re += (-A_re) B_re + A_im B_im ; C_im += (-A_re) B_im + (-A_im) B_re
          lublk::dmma(cr0, cr1, -a0.x, b0.x);
          lublk::dmma(ci0, ci1, -a0.x, b0.y);
          lublk::dmma(cr0, cr1, a0.y, b0.y);
          lublk::dmma(ci0, ci1, -a0.y, b0.x);
          lublk::dmma(cr0, cr1, -a1.x, b1.x);
          lublk::dmma(ci0, ci1, -a1.x, b1.y);
          lublk::dmma(cr0, cr1, a1.y, b1.y);
          lublk::dmma(ci0, ci1, -a1.y, b1.x);
        };
        int tc = r0;
        for (; tc + 8 < NCP; tc += 16) {
          const double2 b0 = A[(kb + bk) * LDA + tc + bcol], b1 = A[(kb + 4 + bk) * LDA + tc + bcol];
          const double2 e0 = A[(kb + bk) * LDA + tc + 8 + bcol], e1 = A[(kb + 4 + bk) * LDA + tc + 8 + bcol];
          double2 *cp = A + (tr + crow) * LDA + tc + ccol;
          const double2 c0 = cp[0], c1 = cp[1], d0 = cp[8], d1 = cp[9];
          double cr0 = c0.x, cr1 = c1.x, ci0 = c0.y, ci1 = c1.y;
          double dr0 = d0.x, dr1 = d1.x, di0 = d0.y, di1 = d1.y;
          tile(cr0, cr1, ci0, ci1, b0, b1);
          tile(dr0, dr1, di0, di1, e0, e1);
          cp[0] = make_double2(cr0, ci0);
          cp[1] = make_double2(cr1, ci1);
          cp[8] = make_double2(dr0, di0);
          cp[9] = make_double2(dr1, di1);
        }
        if (tc < NCP) {
          const double2 b0 = A[(kb + bk) * LDA + tc + bcol], b1 = A[(kb + 4 + bk) * LDA + tc + bcol];
          double2 *cp = A + (tr + crow) * LDA + tc + ccol;
          const double2 c0 = cp[0], c1 = cp[1];
          double cr0 = c0.x, cr1 = c1.x, ci0 = c0.y, ci1 = c1.y;
          tile(cr0, cr1, ci0, ci1, b0, b1);
          cp[0] = make_double2(cr0, ci0);
          cp[1] = make_double2(cr1, ci1);
        }
      }
      __syncwarp();
    }

    LB_TR(2);
    // ---- back substitution U x = y (lane = row), 3 right-hand sides ------------------------------------------------
    double2 *Pw = a.Pws + (size_t)t * 3 * R;
    if (info == 0) {
      double2 y[MS][3];
#pragma unroll
      for (int m = 0; m < MS; ++m) {
        const int i = lane + 32 * m;
#pragma unroll
        for (int c = 0; c < 3; ++c) y[m][c] = (i < R) ? A[i * LDA + R + c] : make_double2(0.0, 0.0);
      }
      double2 ukn[MS];
#pragma unroll
      for (int m = 0; m < MS; ++m) {
        const int i = lane + 32 * m;
        ukn[m] = (i < R - 1) ? A[i * LDA + R - 1] : make_double2(0.0, 0.0);
      }
      double2 rkn = sRinv[R - 1];
#pragma unroll
      for (int mb = MS - 1; mb >= 0; --mb) {
        const int khi = (32 * mb + 31 < R - 1) ? 32 * mb + 31 : R - 1;
#pragma unroll 2
        for (int k = khi; k >= 32 * mb; --k) {
          const double2 rk = rkn;
          double2 uk[MS];
#pragma unroll
          for (int m = 0; m < MS; ++m) uk[m] = ukn[m];
          if (k > 0) {
#pragma unroll
            for (int m = 0; m < MS; ++m) {
              const int i = lane + 32 * m;
              ukn[m] = (i < k - 1) ? A[i * LDA + k - 1] : make_double2(0.0, 0.0);
            }
            rkn = sRinv[k - 1];
          }
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            double2 yk;
            yk.x = __shfl_sync(FULL, y[mb][c].x, k & 31);
            yk.y = __shfl_sync(FULL, y[mb][c].y, k & 31);
            const double2 xk = cmul(yk, rk);
#pragma unroll
            for (int m = 0; m <= mb; ++m) {
              const int i = lane + 32 * m;
              if (i < k) y[m][c] = cfms(uk[m], xk, y[m][c]);
              else if (i == k) y[m][c] = xk;
            }
          }
        }
      }
#pragma unroll
      for (int m = 0; m < MS; ++m) {
        const int i = lane + 32 * m;
        if (i < R) {
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            Pw[c * R + i] = y[m][c];
            if (a.P_out && i < a.r) reinterpret_cast<double2 *>(a.P_out)[((size_t)t * 3 + c) * a.r + i] = y[m][c];
          }
        }
      }
    } else {
      for (int e = lane; e < 3 * R; e += 32) Pw[e] = make_double2(nanv, nanv);
      if (a.P_out)
        for (int e = lane; e < 3 * a.r; e += 32)
          reinterpret_cast<double2 *>(a.P_out)[(size_t)t * 3 * a.r + e] = make_double2(nanv, nanv);
    }
    LB_TR(3);
    if (a.info && lane == 0) a.info[t] = info;
    __syncwarp();
  }
}

template <int R>
static cudaError_t launch_lu_blk_t(const EvalArgs &a, cudaStream_t s) {
  using C = lublk::Cfg<R>;
  auto kern = lu_blk_kernel<R>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::BYTES);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t total = (int64_t)a.n_obj * a.F;
  int64_t blocks = (total + C::WARPS - 1) / C::WARPS;
  if (blocks > sms) blocks = sms;
  kern<<<(unsigned)blocks, C::WARPS * 32, C::BYTES, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_lu_blk(const EvalArgs &a, cudaStream_t s) {
  if (a.flags & PODP_FLAG_NO_PIVOT) return cudaErrorNotSupported;
  switch (a.L.R) {
    case 8: return launch_lu_blk_t<8>(a, s);
    case 16: return launch_lu_blk_t<16>(a, s);
    case 24: return launch_lu_blk_t<24>(a, s);
    case 32: return launch_lu_blk_t<32>(a, s);
    case 40: return launch_lu_blk_t<40>(a, s);
    case 48: return launch_lu_blk_t<48>(a, s);
    case 56: return launch_lu_blk_t<56>(a, s);
    case 64: return launch_lu_blk_t<64>(a, s);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace podp
