// K2 blocked path: panel-blocked right-looking LU with partial pivoting + 3-RHS solve (rows a2-a3).
//   A(omega) = K + i omega nu M,  B(omega) = b0 + omega b1,  P = A^{-1} B            (eqn:ReducedA)
//
// Layout / algorithm.  A group of W warps owns one frequency at a time; [A | B] (R x (R+3) complex, zero-padded
// to R x NCP) lives in the group's slice of shared memory.  Columns are cut into 8-wide tile-columns; tile-column
// c is owned by warp c mod W, which alone applies the row interchanges, forms U12 = L11^{-1} A12 and runs the
// trailing update A22 -= L21 U12 for it -- so warps never wait on each other except for the panel hand-off.
//   * Panel b (tile-column b, rows 8b..R-1) is factored in registers by its owner (lane = row, MS slots) with
//     partial pivoting: redux.sync argmax of an integer magnitude key (lowest row on ties), row interchange and
//     pivot-row broadcast through a 2-row shared scratch, pivot reciprocal by MUFU.RCP64H + 2 Newton steps.
//   * Lookahead: the owner of tile-column b+1 first updates that tile-column with panel b, factors panel b+1 and
//     publishes it (`bar.arrive`, never waits), then updates its other tile-columns; the other warps `bar.sync`.
//   * The trailing update runs on the FP64 tensor path: mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4); a complex 8x8x4
//     product is 4 real DMMAs; C fragments are read/written in shared memory, two tiles interleaved.
//   * B rides along as columns R..R+2 (forward elimination); the factoring warp replaces U11 by its inverse right
//     after publishing a panel, and the back substitution is a left-looking chain of 8x8 DMMA products.
#include <cstdio>
#include <cstdlib>

#include "podp_common.cuh"

namespace podp {

namespace lublk {

constexpr int NB = 8;

template <int R, int W>
struct Cfg {
  static_assert(R % 8 == 0, "R must be a multiple of 8 (exact padding)");
  static constexpr int NCP = R + 8;             // columns incl. RHS block (R..R+2) padded to a tile
  static constexpr int NTC = NCP / 8;           // tile-columns
  static constexpr int LDA = NCP + 1;           // row stride (complex), odd: 16-byte-bank rotation per row
  static constexpr int MS = (R + 31) / 32;      // panel row slots per lane
  static constexpr int A_ELEMS = R * LDA;
  static constexpr int G_BYTES = A_ELEMS * 16 + R * 16 + 2 * NB * 16 + R * 4 + 16;  // A, 1/U_kk, scratch, pivots
  static constexpr int GROUPS_SMEM = (225 * 1024) / G_BYTES;
  // <= 16 warps per CTA; with W > 1 each group uses 3 named barriers (ids 1..15 available)
  static constexpr int GROUPS_T = W == 1 ? 16 : ((16 / W) < 5 ? (16 / W) : 5);
  static constexpr int GROUPS = GROUPS_SMEM < GROUPS_T ? GROUPS_SMEM : GROUPS_T;
  static constexpr int THREADS = GROUPS * W * 32;
  static constexpr size_t BYTES = (size_t)GROUPS * G_BYTES;
  static_assert(GROUPS >= 1, "matrix does not fit in shared memory");
};

__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// The inverse of the upper-triangular diagonal block U11 of a factored panel replaces U11 in place (its slots are
// dead: the trailing updates use L11, L21 and U12 only).  Lane -> (block kb0 + 8 (lane / 8), column lane % 8), nblk
// <= 4 blocks per call; column c comes from back substitution with 1/U_kk from sRinv; all loads precede all writes.
template <int LDA>
__device__ __forceinline__ void invert_diag(double2 *A, const double2 *sRinv, int kb0, int nblk, int lane) {
  constexpr int NB = 8;
  double2 x[NB];
  const bool act = lane < NB * nblk;
  const int kb = kb0 + NB * (lane >> 3), c = lane & 7;
  if (act) {
#pragma unroll
    for (int j = NB - 1; j >= 0; --j) {
      const double2 rj = sRinv[kb + j];
      double2 acc = make_double2(0.0, 0.0);
#pragma unroll
      for (int t = j + 1; t < NB; ++t) acc = cfma(A[(kb + j) * LDA + kb + t], x[t], acc);
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

}  // namespace lublk

template <int R, int W>
__global__ void __launch_bounds__(lublk::Cfg<R, W>::THREADS, 1) lu_blk_kernel(EvalArgs a) {
  using C = lublk::Cfg<R, W>;
  constexpr int NCP = C::NCP, NTC = C::NTC, LDA = C::LDA, MS = C::MS, NB = lublk::NB, NT = W * 32;
  constexpr int NPAN = R / NB;
  // U11^{-1} in place right after each panel is published (in the factoring warp's slack) or, where that slack is
  // too short (W = 1, and the two-warp R = 48 case, measured), for all blocks just before the back substitution
  constexpr bool INV_EARLY = W > 1 && !(W == 2 && R == 48);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = wid / W, w = wid % W;
  unsigned char *gbase = smem_raw + (size_t)grp * C::G_BYTES;
  double2 *A = reinterpret_cast<double2 *>(gbase);
  double2 *sRinv = A + C::A_ELEMS;
  double2 *sRowK = sRinv + R, *sRowP = sRowK + NB;  // panel scratch rows (old row k, pivot row)
  int *sPiv = reinterpret_cast<int *>(sRowP + NB);  // [R] pivots, [R] group status
  const int bar0 = 1 + 3 * grp;  // ids bar0, bar0+1 (alternating panel hand-offs), bar0+2 (full group)
  const int64_t total = (int64_t)a.n_obj * a.F;
  const double nanv = __longlong_as_double(0x7ff8000000000000ll);
  const unsigned FULL = 0xffffffffu;
  const int ngroups_total = gridDim.x * C::GROUPS;
  (void)NCP;

  // ---- panel factorisation of tile-column b by the calling warp (sets info != 0 on a zero pivot) -------------
  // Rows never move inside the panel: lane owns the panel rows loaded from positions kb + lane + 32 m and tracks
  // each row's current position (LAPACK interchange semantics).  The pivot search key carries the POSITION, so
  // ties resolve to the lowest position as in izamax; only the pivot row is broadcast (8 values via smem).
  auto factor_panel = [&](int b, int &info) __attribute__((always_inline)) {
    const int kb = b * NB;
    double2 pn[MS][NB];
    int pos[MS];
#pragma unroll
    for (int m = 0; m < MS; ++m) {
      const int i = kb + lane + 32 * m;
      pos[m] = i < R ? i : 1 << 20;
#pragma unroll
      for (int c = 0; c < NB; ++c) pn[m][c] = (i < R) ? A[i * LDA + kb + c] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      const int kr = kb + j;
      unsigned key = 0u;
#pragma unroll
      for (int m = 0; m < MS; ++m) {
        const unsigned kk = (mag_key_hi(pn[m][j]) & 0xFFFFFF80u) | (unsigned)(127 - pos[m]);
        if (pos[m] >= kr && pos[m] < R && kk > key) key = kk;
      }
      const unsigned best = __reduce_max_sync(FULL, key);
      if ((best >> 7) == 0u) {
        if (info == 0) info = kr + 1;
        return;
      }
      const int p = 127 - (int)(best & 127u);  // pivot position
      // the row now at position p is the pivot row: broadcast its panel values; positions kr <-> p swap
      bool mine[MS];
#pragma unroll
      for (int m = 0; m < MS; ++m) {
        mine[m] = pos[m] == p;
        if (mine[m]) {
#pragma unroll
          for (int c = j; c < NB; ++c) sRowP[c] = pn[m][c];
        }
      }
      if (lane == 0) sPiv[kr] = p;
      __syncwarp();
      const double2 pv = sRowP[j];
      double2 u[NB];
#pragma unroll
      for (int c = j + 1; c < NB; ++c) u[c] = sRowP[c];
#pragma unroll
      for (int m = 0; m < MS; ++m) pos[m] = mine[m] ? kr : (pos[m] == kr ? p : pos[m]);
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
      __syncwarp();  // scratch row reused by the next column
    }
    // write the factored panel back at the rows' final positions (L21 multipliers, U11)
#pragma unroll
    for (int m = 0; m < MS; ++m) {
      if (pos[m] < R) {
#pragma unroll
        for (int c = 0; c < NB; ++c) A[pos[m] * LDA + kb + c] = pn[m][c];
      }
    }
  };

  // ---- apply panel b (interchanges, U12, trailing update) to tile-column tcol (owned by the calling warp) -------
  auto update_tile_col = [&](int b, int tcol) __attribute__((always_inline)) {
    const int kb = b * NB;
    const int col0 = tcol * 8;
    // (1) interchanges + U12 = L11^{-1} A12: lanes 0..7 own one column each
    if (lane < 8) {
      const int col = col0 + lane;
      double2 x[NB];
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        const int p = sPiv[kb + j];
        const double2 vk = A[(kb + j) * LDA + col];
        if (p != kb + j) {
          x[j] = A[p * LDA + col];
          A[p * LDA + col] = vk;
        } else {
          x[j] = vk;
        }
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
    // (2) A22[:, tile] -= L21 U12[:, tile] on 8x8 complex tiles; two row-tiles interleaved
    const int arow = lane >> 2, acol = lane & 3;
    const int bk = lane & 3, bcol = lane >> 2;
    const int crow = lane >> 2, ccol = 2 * (lane & 3);
    const double2 b0 = A[(kb + bk) * LDA + col0 + bcol], b1 = A[(kb + 4 + bk) * LDA + col0 + bcol];
    auto tile = [&](double &cr0, double &cr1, double &ci0, double &ci1, double2 a0, double2 a1)
        __attribute__((always_inline)) {
      // C -= A B (complex): C_re += (-A_re) B_re + A_im B_im ; C_im += (-A_re) B_im + (-A_im) B_re
      lublk::dmma(cr0, cr1, -a0.x, b0.x);
      lublk::dmma(ci0, ci1, -a0.x, b0.y);
      lublk::dmma(cr0, cr1, a0.y, b0.y);
      lublk::dmma(ci0, ci1, -a0.y, b0.x);
      lublk::dmma(cr0, cr1, -a1.x, b1.x);
      lublk::dmma(ci0, ci1, -a1.x, b1.y);
      lublk::dmma(cr0, cr1, a1.y, b1.y);
      lublk::dmma(ci0, ci1, -a1.y, b1.x);
    };
    int tr = kb + NB;
    for (; tr + 8 < R; tr += 16) {
      const double2 a0 = A[(tr + arow) * LDA + kb + acol], a1 = A[(tr + arow) * LDA + kb + 4 + acol];
      const double2 e0 = A[(tr + 8 + arow) * LDA + kb + acol], e1 = A[(tr + 8 + arow) * LDA + kb + 4 + acol];
      double2 *cp = A + (tr + crow) * LDA + col0 + ccol;
      double2 *dp = cp + 8 * LDA;
      const double2 c0 = cp[0], c1 = cp[1], d0 = dp[0], d1 = dp[1];
      double cr0 = c0.x, cr1 = c1.x, ci0 = c0.y, ci1 = c1.y;
      double dr0 = d0.x, dr1 = d1.x, di0 = d0.y, di1 = d1.y;
      tile(cr0, cr1, ci0, ci1, a0, a1);
      tile(dr0, dr1, di0, di1, e0, e1);
      cp[0] = make_double2(cr0, ci0);
      cp[1] = make_double2(cr1, ci1);
      dp[0] = make_double2(dr0, di0);
      dp[1] = make_double2(dr1, di1);
    }
    if (tr < R) {
      const double2 a0 = A[(tr + arow) * LDA + kb + acol], a1 = A[(tr + arow) * LDA + kb + 4 + acol];
      double2 *cp = A + (tr + crow) * LDA + col0 + ccol;
      const double2 c0 = cp[0], c1 = cp[1];
      double cr0 = c0.x, cr1 = c1.x, ci0 = c0.y, ci1 = c1.y;
      tile(cr0, cr1, ci0, ci1, a0, a1);
      cp[0] = make_double2(cr0, ci0);
      cp[1] = make_double2(cr1, ci1);
    }
    __syncwarp();
  };

  for (int64_t t = (int64_t)blockIdx.x * C::GROUPS + grp; t < total; t += ngroups_total) {
    const int obj = (int)(t / a.F);
    const int64_t f = t - (int64_t)obj * a.F;
    const double *op = a.ops + (size_t)obj * a.L.stride;
    const double om = a.omega[f];
    const double s = om * op[a.L.scal + SC_NU];
    // ---- a2: assemble [A | B | 0] (all W warps).  K and M stream through registers in batches (all loads of a
    //      batch in flight at once) and A = K + i s M is written to shared memory once (one pass of shared-memory
    //      traffic per element instead of the copy + read-modify-write of a cp.async assembly). -----------------
    {
      const double2 *gK = reinterpret_cast<const double2 *>(op + a.L.K);
      const double2 *gM = reinterpret_cast<const double2 *>(op + a.L.M);
      constexpr int PER = (R * R + NT - 1) / NT;
      constexpr int BAT = PER < 12 ? PER : 12;  // elements per batch and thread
      const int gl = w * 32 + lane;
      const double2 *gb0 = reinterpret_cast<const double2 *>(op + a.L.b0);
      const double2 *gb1 = reinterpret_cast<const double2 *>(op + a.L.b1);
#pragma unroll
      for (int q = 0; q < (8 * R + NT - 1) / NT; ++q) {
        const int e = q * NT + gl;
        if (e >= 8 * R) break;
        const int i = e >> 3, c = e & 7;
        double2 v = make_double2(0.0, 0.0);
        if (c < 3) {
          const double2 x0 = __ldg(gb0 + c * R + i), x1 = __ldg(gb1 + c * R + i);
          v = make_double2(fma(om, x1.x, x0.x), fma(om, x1.y, x0.y));
        }
        A[i * LDA + R + c] = v;
      }
#pragma unroll
      for (int q0 = 0; q0 < PER; q0 += BAT) {
        double2 kk[BAT], mm[BAT];
#pragma unroll
        for (int q = 0; q < BAT; ++q) {
          const int e = (q0 + q) * NT + gl;
          if (q0 + q < PER && e < R * R) {
            kk[q] = __ldg(gK + e);
            mm[q] = __ldg(gM + e);
          }
        }
#pragma unroll
        for (int q = 0; q < BAT; ++q) {
          const int e = (q0 + q) * NT + gl;
          if (q0 + q < PER && e < R * R) {
            const int i = e / R, j = e - i * R;
            A[i * LDA + j] = make_double2(fma(-s, mm[q].y, kk[q].x), fma(s, mm[q].x, kk[q].y));
          }
        }
      }
    }
    if constexpr (W > 1) lublk::bar_sync(bar0 + 2, NT); else __syncwarp();
    int info = isfinite(om) ? 0 : -1;
    // ---- a3: blocked LU -- panel 0 by its owner (warp 0); group status lives in sPiv[R] ---------------------------
    if (w == 0) {
      if (info == 0) factor_panel(0, info);
      if (lane == 0) sPiv[R] = info;
      __syncwarp();
      if constexpr (W > 1) {
        lublk::bar_arrive(bar0, NT);
        if (INV_EARLY && info == 0) lublk::invert_diag<LDA>(A, sRinv, 0, 1, lane);  // off the critical chain
      }
    }
    for (int b = 0; b < NPAN; ++b) {
      const int owner = b % W;
      if constexpr (W > 1) {
        if (w != owner) lublk::bar_sync(bar0 + (b & 1), NT);
      } else {
        __syncwarp();
      }
      info = sPiv[R];
      const bool next = b + 1 < NPAN;
      const int nowner = (b + 1) % W;
      bool inv_next = false;
      if (info == 0 && next && w == nowner) {
        // lookahead: the owner of tile-column b+1 updates it, factors panel b+1 and publishes it
        update_tile_col(b, b + 1);
        int inf2 = 0;
        factor_panel(b + 1, inf2);
        if (lane == 0) sPiv[R] = inf2;
        __syncwarp();
        inv_next = inf2 == 0;
      }
      if (next && w == nowner) {
        if constexpr (W > 1) {
          lublk::bar_arrive(bar0 + ((b + 1) & 1), NT);
          if (INV_EARLY && inv_next) lublk::invert_diag<LDA>(A, sRinv, (b + 1) * NB, 1, lane);  // off the chain
        }
      }
      if (info == 0) {
        for (int tc = b + 1; tc < NTC; ++tc) {
          if (tc % W != w) continue;
          if (next && tc == b + 1) continue;  // done in the lookahead
          update_tile_col(b, tc);
        }
      }
    }
    if constexpr (W > 1) lublk::bar_sync(bar0 + 2, NT); else __syncwarp();
    info = sPiv[R];
    // ---- back substitution U x = y, blocked and left-looking on the FP64 tensor path (warp 0).  The inverses
    //      Dinv_b of the diagonal blocks were formed in place of U11 by the factoring warps (INV_EARLY) or are formed
    //      here; for b = NPAN-1 .. 0: y_b -= sum_{b' > b} U_{b b'} x_{b'} (DMMA, two accumulators), x_b = Dinv_b y_b.
    //      The right-hand-side tile (8 columns, 3 used) is the DMMA n dimension.
    double2 *Pw = a.Pws + (size_t)t * 3 * R;
    if constexpr (!INV_EARLY) {
      if (info == 0) {  // every warp inverts up to 4 diagonal blocks (warp w: blocks 4w ..), then one hand-off
        for (int b0 = 4 * w; b0 < NPAN; b0 += 4 * W)
          lublk::invert_diag<LDA>(A, sRinv, b0 * NB, NPAN - b0 < 4 ? NPAN - b0 : 4, lane);
        if constexpr (W > 1) lublk::bar_sync(bar0 + 2, NT);
      }
    }
    if (w == 0) {
      if (info == 0) {
        const int arow = lane >> 2, acol = lane & 3;
        const int bk = lane & 3, bcol = lane >> 2;
        const int crow = lane >> 2, ccol = 2 * (lane & 3);
        for (int b = NPAN - 1; b >= 0; --b) {
          const int kb = b * 8;
          double2 y0 = A[(kb + crow) * LDA + R + ccol], y1 = A[(kb + crow) * LDA + R + ccol + 1];
          double cr0 = y0.x, cr1 = y1.x, ci0 = y0.y, ci1 = y1.y;
          double dr0 = 0.0, dr1 = 0.0, di0 = 0.0, di1 = 0.0;
#pragma unroll
          for (int d = 1; d < NPAN; ++d) {
            const int bb = b + d;
            if (bb >= NPAN) break;
            const int kc = bb * 8;
            const double2 a0 = A[(kb + arow) * LDA + kc + acol], a1 = A[(kb + arow) * LDA + kc + 4 + acol];
            const double2 x0 = A[(kc + bk) * LDA + R + bcol], x1 = A[(kc + 4 + bk) * LDA + R + bcol];
            if (d & 1) {
              lublk::dmma(cr0, cr1, -a0.x, x0.x);
              lublk::dmma(ci0, ci1, -a0.x, x0.y);
              lublk::dmma(cr0, cr1, a0.y, x0.y);
              lublk::dmma(ci0, ci1, -a0.y, x0.x);
              lublk::dmma(cr0, cr1, -a1.x, x1.x);
              lublk::dmma(ci0, ci1, -a1.x, x1.y);
              lublk::dmma(cr0, cr1, a1.y, x1.y);
              lublk::dmma(ci0, ci1, -a1.y, x1.x);
            } else {
              lublk::dmma(dr0, dr1, -a0.x, x0.x);
              lublk::dmma(di0, di1, -a0.x, x0.y);
              lublk::dmma(dr0, dr1, a0.y, x0.y);
              lublk::dmma(di0, di1, -a0.y, x0.x);
              lublk::dmma(dr0, dr1, -a1.x, x1.x);
              lublk::dmma(di0, di1, -a1.x, x1.y);
              lublk::dmma(dr0, dr1, a1.y, x1.y);
              lublk::dmma(di0, di1, -a1.y, x1.x);
            }
          }
          __syncwarp();
          A[(kb + crow) * LDA + R + ccol] = make_double2(cr0 + dr0, ci0 + di0);
          A[(kb + crow) * LDA + R + ccol + 1] = make_double2(cr1 + dr1, ci1 + di1);
          __syncwarp();
          // x_b = Dinv_b y_b (Dinv_b stored in place of U11)
          const int m = arow, k0 = acol, k1 = acol + 4;
          const double2 v0 = m <= k0 ? A[(kb + m) * LDA + kb + k0] : make_double2(0.0, 0.0);
          const double2 v1 = m <= k1 ? A[(kb + m) * LDA + kb + k1] : make_double2(0.0, 0.0);
          const double2 x0 = A[(kb + bk) * LDA + R + bcol], x1 = A[(kb + 4 + bk) * LDA + R + bcol];
          double er0 = 0.0, er1 = 0.0, ei0 = 0.0, ei1 = 0.0;
          lublk::dmma(er0, er1, v0.x, x0.x);
          lublk::dmma(ei0, ei1, v0.x, x0.y);
          lublk::dmma(er0, er1, -v0.y, x0.y);
          lublk::dmma(ei0, ei1, v0.y, x0.x);
          lublk::dmma(er0, er1, v1.x, x1.x);
          lublk::dmma(ei0, ei1, v1.x, x1.y);
          lublk::dmma(er0, er1, -v1.y, x1.y);
          lublk::dmma(ei0, ei1, v1.y, x1.x);
          __syncwarp();
          A[(kb + crow) * LDA + R + ccol] = make_double2(er0, ei0);
          A[(kb + crow) * LDA + R + ccol + 1] = make_double2(er1, ei1);
          __syncwarp();
        }
        for (int e = lane; e < 3 * R; e += 32) {
          const int c = e / R, i = e - c * R;
          const double2 v = A[i * LDA + R + c];
          Pw[e] = v;
          if (a.P_out && i < a.r) reinterpret_cast<double2 *>(a.P_out)[((size_t)t * 3 + c) * a.r + i] = v;
        }
      } else {
        for (int e = lane; e < 3 * R; e += 32) Pw[e] = make_double2(nanv, nanv);
        if (a.P_out)
          for (int e = lane; e < 3 * a.r; e += 32)
            reinterpret_cast<double2 *>(a.P_out)[(size_t)t * 3 * a.r + e] = make_double2(nanv, nanv);
      }
    }
    if (a.info && w == 0 && lane == 0) a.info[t] = info;
    if constexpr (W > 1) lublk::bar_sync(bar0 + 2, NT); else __syncwarp();
  }
}

template <int R, int W>
static cudaError_t launch_lu_blk_t(const EvalArgs &a, cudaStream_t s) {
  using C = lublk::Cfg<R, W>;
  auto kern = lu_blk_kernel<R, W>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::BYTES);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t total = (int64_t)a.n_obj * a.F;
  int64_t blocks = (total + C::GROUPS - 1) / C::GROUPS;
  if (blocks > sms) blocks = sms;
  kern<<<(unsigned)blocks, C::THREADS, C::BYTES, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_lu_blk(const EvalArgs &a, cudaStream_t s) {
  if (a.flags & PODP_FLAG_NO_PIVOT) return cudaErrorNotSupported;
  // measured on B200 (tools/r_sweep.py): one warp per frequency is best for r <= 32, two for r = 40..56, four for
  // r = 64..72, eight for r >= 80 (shared memory then holds a single frequency per SM)
  const int wv = (a.L.R >= 80 ? 8 : (a.L.R >= 64 ? 4 : (a.L.R >= 40 ? 2 : 1)));
  switch (a.L.R) {
#define PODP_CASE(RR)                                 \
  case RR:                                            \
    if (wv == 1) return launch_lu_blk_t<RR, 1>(a, s); \
    if (wv == 2) return launch_lu_blk_t<RR, 2>(a, s); \
    if (wv == 8 && RR >= 64) return launch_lu_blk_t<(RR >= 64 ? RR : 64), 8>(a, s); \
    return launch_lu_blk_t<RR, 4>(a, s);
    PODP_CASE(8)
    PODP_CASE(16)
    PODP_CASE(24)
    PODP_CASE(32)
    PODP_CASE(40)
    PODP_CASE(48)
    PODP_CASE(56)
    PODP_CASE(64)
    PODP_CASE(72)
    PODP_CASE(80)
    PODP_CASE(88)
    PODP_CASE(96)
#undef PODP_CASE
    default: return cudaErrorNotSupported;
  }
}

}  // namespace podp
