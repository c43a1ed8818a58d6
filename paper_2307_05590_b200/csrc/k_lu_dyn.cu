// K2 default path: batched shifted complex LU with partial pivoting + 3-RHS solve, dynamically scheduled (rows a2-a3).
//   A(omega) = K + i omega nu M,  B(omega) = b0 + omega b1,  P = A^{-1} B            (eqn:ReducedA)
//   "the cost of solving (eqn:ReducedA) is at most O(M^3)": this kernel is that O(r^3) step.
//
// One group of W warps owns one frequency at a time; [A | B] (R x (R+3) complex, zero-padded to R x (R+8)) lives in
// the group's slice of shared memory.  The columns are cut into 8-wide tile-columns; tile-column c belongs to warp
// c mod W.  Two kinds of task exist:
//   F(k)     factor panel k (tile-column k, rows 8k..R-1) with partial pivoting -- in registers, one warp, lane = row;
//            the pivot search is one redux.sync over an integer magnitude key, the pivot row is broadcast by
//            shuffles (no shared-memory round trip on the per-column chain), 1/pivot is MUFU.RCP64H + 2 Newton steps.
//            Rows never move inside the panel; the panel is written back at the rows' final positions together with
//            the step's permutation (orig[] / dst[]), then published (release store of a counter in shared memory).
//   U(k, c)  apply panel k to tile-column c: permute the column in one pass (the 8 pivot rows in, the displaced rows
//            out), U12 = L11^{-1} A12 (8 lanes, one column each), A22 -= L21 U12 on the FP64 tensor path
//            (mma.sync.m8n8k4.f64 = DMMA; a complex 8x8x4 product is 4 real DMMAs), loads of a chunk of row tiles
//            issued before its DMMAs.
// Each warp runs its own task loop with no lock-step barriers: first the critical chain (bring its next panel up to
// date and factor it as soon as the panels it needs are published), then the oldest ready backlog update, else it
// polls the publish counter.  This is a lookahead of arbitrary depth: a panel is factored as soon as its column is
// current, and the rest of the trailing update fills the gaps.
// L is never stored for later use: B rides along as columns R..R+2, so forward elimination happens in the updates
// and only U remains for the back substitution, which runs on one warp with the solution in registers (lane = row).
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "lu_tasks.cuh"

namespace podp {

namespace ludyn {

constexpr int NB = 8;

// RG: the right-hand-side tile and the pivot reciprocals live in a per-group L2-resident scratch instead of shared
// memory, which lets one more group fit per SM where A alone is just small enough (r = 48: 6 instead of 5).
template <int R, int W, bool RG = false>
struct Cfg {
  static_assert(R % 8 == 0, "R must be a multiple of 8 (exact padding)");
  static constexpr int NPAN = R / NB;           // panels
  static constexpr int NCP = RG ? R : R + 8;    // shared-memory columns (+ the RHS tile R..R+7 unless RG)
  static constexpr int NTC = NPAN + 1;          // tile-columns incl. the right-hand-side tile
  static constexpr int LDA = NCP + 1;           // row stride (complex), odd
  static constexpr int MS = (R + 31) / 32;      // panel row slots per lane
  static constexpr int NOWN = (NTC + W - 1) / W;  // tile-columns per warp (upper bound)
  static constexpr int A_ELEMS = R * LDA;
  // A, 1/U_kk (R), orig (R), dst (R), {published panels, info, pad}, pivot-row scratch (9)
  // ... + one mbarrier per panel (completes when the panel is published)
  // (rounded to 16 B so that every group's base stays aligned)
  static constexpr int G_BYTES = (A_ELEMS * 16 + (RG ? 0 : R * 16) + 2 * R * 4 + 16 + 9 * 16 + NPAN * 8 + 15) / 16 * 16;
  static constexpr int GROUPS_SMEM = (227 * 1024) / G_BYTES;
  static constexpr int GROUPS_T = (16 / W) < 15 ? (16 / W) : 15;  // <= 16 warps, one named barrier per group
  static constexpr int GROUPS = GROUPS_SMEM < GROUPS_T ? GROUPS_SMEM : GROUPS_T;
  static constexpr int THREADS = GROUPS * W * 32;
  static constexpr size_t BYTES = (size_t)GROUPS * G_BYTES;
  static_assert(GROUPS >= 1, "matrix does not fit in shared memory");
};

__device__ __forceinline__ void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void mbar_init(unsigned long long *m, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(m)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long *m) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.release.cta.shared::cta.b64 st, [%0];\n\t}" ::"r"(
                   (unsigned)__cvta_generic_to_shared(m))
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(unsigned long long *m, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"((unsigned)__cvta_generic_to_shared(m)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ int ld_acquire(const int *p) {
  int v;
  asm volatile("ld.acquire.cta.shared.b32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int *p, int v) {
  asm volatile("st.release.cta.shared.b32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(p)), "r"(v) : "memory");
}
}  // namespace ludyn



template <int R, int W, bool RG>
__global__ void __launch_bounds__(ludyn::Cfg<R, W, RG>::THREADS, 1) lu_dyn_kernel(EvalArgs a) {
  using C = ludyn::Cfg<R, W, RG>;
  constexpr int NTC = C::NTC, LDA = C::LDA, MS = C::MS, NB = ludyn::NB, NT = W * 32, NPAN = C::NPAN;
  constexpr int NOWN = C::NOWN;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = wid / W, w = wid % W;
  unsigned char *gbase = smem_raw + (size_t)grp * C::G_BYTES;
  double2 *A = reinterpret_cast<double2 *>(gbase);
  // RG: per-group scratch in L2: RHS tile (R x 8, row stride 8) then 1/U_kk (R)
  double2 *gRHS = RG ? a.gscr + ((size_t)blockIdx.x * C::GROUPS + grp) * (9 * R) : nullptr;
  double2 *sRinv = RG ? gRHS + 8 * R : A + C::A_ELEMS;
  int *sOrig = reinterpret_cast<int *>(A + C::A_ELEMS + (RG ? 0 : R));  // pre-step position of the row now at q
  int *sDst = sOrig + R;                             // sDst[o]: final position of the row that was at o (o in panel)
  int *sPub = sDst + R;                              // [0] panels published, [1] info
  double2 *sRow = reinterpret_cast<double2 *>(sPub + 4);  // pivot-row scratch (8 values + position)
  unsigned long long *sBar = reinterpret_cast<unsigned long long *>(sRow + 9);  // [NPAN] publish mbarriers
  if (w == 0 && lane == 0)
    for (int k = 0; k < NPAN; ++k) ludyn::mbar_init(sBar + k, 1);
  __syncthreads();
  unsigned lu_par = 0;  // phase parity of the publish mbarriers (flips once per factorised frequency)
  const int bar_id = 1 + grp;
  const int64_t total = (int64_t)a.n_obj * a.F;
  const double nanv = __longlong_as_double(0x7ff8000000000000ll);
  const int ngroups_total = gridDim.x * C::GROUPS;

  for (int64_t t = (int64_t)blockIdx.x * C::GROUPS + grp; t < total; t += ngroups_total) {
    const int obj = (int)(t / a.F);
    const int64_t f = t - (int64_t)obj * a.F;
    const double *op = a.ops + (size_t)obj * a.L.stride;
    const double om = a.omega[f];
    const double s = om * op[a.L.scal + SC_NU];
    // ---- a2: assemble [A | B | 0] (all W warps).  K and M stream through registers in batches (all loads of a
    //      batch in flight at once) and A = K + i s M is written to shared memory once. -----------------------------
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
        if constexpr (RG) gRHS[i * 8 + c] = v; else A[i * LDA + R + c] = v;
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
      if (w == 0 && lane == 0) {
        sPub[0] = 0;
        sPub[1] = isfinite(om) ? 0 : -1;
      }
    }
    if constexpr (W > 1) ludyn::bar_sync(bar_id, NT); else __syncwarp();
    // ---- a3: dynamically scheduled blocked LU ------------------------------------------------------------------------
    // every warp derives the LU's go/no-go from omega itself: sPub[1] may already carry a zero-pivot info written
    // by a warp that started factoring (data race on the shared status word)
    const bool lu_run = isfinite(om);
    if (lu_run) {
      int done[NOWN];  // updates applied to each owned tile-column (tile w + q W)
#pragma unroll
      for (int q = 0; q < NOWN; ++q) done[q] = 0;
      int nf = w;       // next panel this warp factors (tile index; >= NPAN: none left)
      int pub = 0;      // panels known to be published
      unsigned spins = 0;
      for (;;) {
        // pick the next task: (1) the critical chain -- bring the next own panel up to date and factor it;
        // (2) else the owned tile-column with the fewest applied panels among the ready ones; (3) else poll.
        int ub = -1, uq = -1;  // update task U(ub, tile w + uq W)
        if (nf < NPAN) {
          int dn = 0, qn = 0;
#pragma unroll
          for (int q = 0; q < NOWN; ++q)
            if (w + q * W == nf) {
              dn = done[q];
              qn = q;
            }
          if (dn == nf) {
            const int inf = (R - nf * NB > 32)
                                ? ludyn::factor_panel<R, LDA, MS>(A, sRinv, sOrig, sDst, sRow, nf * NB, lane)
                                : ludyn::factor_panel<R, LDA, 1>(A, sRinv, sOrig, sDst, sRow, nf * NB, lane);
            __threadfence_block();
            __syncwarp();
            if (lane == 0) {
              if (inf != 0 && sPub[1] == 0) sPub[1] = inf;
              ludyn::st_release(sPub, nf + 1);
              ludyn::mbar_arrive(sBar + nf);
            }
            if (nf + 1 > pub) pub = nf + 1;
            // W > 1: invert U11 now, in the slack before this warp's next critical task; W = 1 does all blocks at the end
            if constexpr (W > 1)
              if (inf == 0) ludyn::invert_diag<LDA>(A, sRinv, nf * NB, 1, lane);
            nf += W;
            continue;
          }
          if (dn >= pub) pub = ludyn::ld_acquire(sPub);
          if (dn < pub) {
            ub = dn;
            uq = qn;
          }
        }
        if (uq < 0) {
          int best_d = 1 << 20;
          bool all = nf >= NPAN;
#pragma unroll
          for (int q = 0; q < NOWN; ++q) {
            const int tc = w + q * W;
            if (tc < NTC) {
              const int lim = tc < NPAN ? tc : NPAN;
              if (done[q] < lim) {
                all = false;
                if (!(nf < NPAN && tc == nf) && done[q] < pub && done[q] < best_d) {
                  best_d = done[q];
                  uq = q;
                }
              }
            }
          }
          if (all) break;
          if (uq < 0) {
            // nothing ready: block (hardware-suspended try_wait) until the next panel is published
            while (!ludyn::mbar_try_wait(sBar + pub, lu_par))
              if (++spins > (1 << 24)) __trap();  // scheduling invariant broken: fail loudly instead of hanging
            pub = ludyn::ld_acquire(sPub);
            continue;
          }
          ub = best_d;
        }
        {
          const int tcu = w + uq * W;
          if (RG && tcu == NPAN)
            ludyn::update_dispatch<R, LDA, 8>(A, gRHS, sOrig, sDst, ub, lane);
          else
            ludyn::update_dispatch<R, LDA, LDA>(A, A + tcu * 8, sOrig, sDst, ub, lane);
        }
#pragma unroll
        for (int q = 0; q < NOWN; ++q)
          if (q == uq) done[q] += 1;
      }
    }
    {
      if constexpr (W > 1) ludyn::bar_sync(bar_id, NT); else __syncwarp();
    }
    if (lu_run) lu_par ^= 1u;
    const int info = sPub[1];
    // ---- back substitution U x = y, blocked and left-looking on the FP64 tensor path.
    //      The inverses Dinv_b of the diagonal blocks were formed in place by the factoring warps (invert_diag);
    //      warp 0, for b = NPAN-1 .. 0: y_b -= sum_{b' > b} U_{b b'} x_{b'} (DMMA, two accumulators), then
    //      x_b = Dinv_b y_b (DMMA).  The right-hand-side tile (8 columns, 3 used) is the DMMA n dimension.
    double2 *Pw = a.Pws + (size_t)t * 3 * R;
    if (w == 0) {
      if (info == 0) {
        if constexpr (W == 1) {
#pragma unroll
          for (int b0 = 0; b0 < NPAN; b0 += 4)
            ludyn::invert_diag<LDA>(A, sRinv, b0 * NB, NPAN - b0 < 4 ? NPAN - b0 : 4, lane);
        }
        const int arow = lane >> 2, acol = lane & 3;
        const int bk = lane & 3, bcol = lane >> 2;
        const int crow = lane >> 2, ccol = 2 * (lane & 3);
        if constexpr (RG) {
          // y prefetched from the L2 scratch once; x kept as B fragments in registers (C -> B by shuffles); the
          // solution goes straight from the C fragments to the hand-off workspace
          double2 ya[NPAN], yb[NPAN], xb0[NPAN], xb1[NPAN];
#pragma unroll
          for (int b = 0; b < NPAN; ++b) {
            ya[b] = gRHS[(8 * b + crow) * 8 + ccol];
            yb[b] = gRHS[(8 * b + crow) * 8 + ccol + 1];
          }
#pragma unroll
          for (int b = NPAN - 1; b >= 0; --b) {
            const int kb = b * 8;
            double cr0 = ya[b].x, cr1 = yb[b].x, ci0 = ya[b].y, ci1 = yb[b].y;
            double dr0 = 0.0, dr1 = 0.0, di0 = 0.0, di1 = 0.0;
#pragma unroll
            for (int bb = b + 1; bb < NPAN; ++bb) {
              const int kc = bb * 8;
              const double2 a0 = A[(kb + arow) * LDA + kc + acol], a1 = A[(kb + arow) * LDA + kc + 4 + acol];
              const double2 x0 = xb0[bb], x1 = xb1[bb];
              if ((bb - b) & 1) {
                ludyn::dmma(cr0, cr1, -a0.x, x0.x);
                ludyn::dmma(ci0, ci1, -a0.x, x0.y);
                ludyn::dmma(cr0, cr1, a0.y, x0.y);
                ludyn::dmma(ci0, ci1, -a0.y, x0.x);
                ludyn::dmma(cr0, cr1, -a1.x, x1.x);
                ludyn::dmma(ci0, ci1, -a1.x, x1.y);
                ludyn::dmma(cr0, cr1, a1.y, x1.y);
                ludyn::dmma(ci0, ci1, -a1.y, x1.x);
              } else {
                ludyn::dmma(dr0, dr1, -a0.x, x0.x);
                ludyn::dmma(di0, di1, -a0.x, x0.y);
                ludyn::dmma(dr0, dr1, a0.y, x0.y);
                ludyn::dmma(di0, di1, -a0.y, x0.x);
                ludyn::dmma(dr0, dr1, -a1.x, x1.x);
                ludyn::dmma(di0, di1, -a1.x, x1.y);
                ludyn::dmma(dr0, dr1, a1.y, x1.y);
                ludyn::dmma(di0, di1, -a1.y, x1.x);
              }
            }
            double2 y0b, y1b;
            ludyn::c_to_b(make_double2(cr0 + dr0, ci0 + di0), make_double2(cr1 + dr1, ci1 + di1), lane, y0b, y1b);
            const int m = arow, k0 = acol, k1 = acol + 4;
            const double2 v0 = m <= k0 ? A[(kb + m) * LDA + kb + k0] : make_double2(0.0, 0.0);
            const double2 v1 = m <= k1 ? A[(kb + m) * LDA + kb + k1] : make_double2(0.0, 0.0);
            double er0 = 0.0, er1 = 0.0, ei0 = 0.0, ei1 = 0.0;
            ludyn::dmma(er0, er1, v0.x, y0b.x);
            ludyn::dmma(ei0, ei1, v0.x, y0b.y);
            ludyn::dmma(er0, er1, -v0.y, y0b.y);
            ludyn::dmma(ei0, ei1, v0.y, y0b.x);
            ludyn::dmma(er0, er1, v1.x, y1b.x);
            ludyn::dmma(ei0, ei1, v1.x, y1b.y);
            ludyn::dmma(er0, er1, -v1.y, y1b.y);
            ludyn::dmma(ei0, ei1, v1.y, y1b.x);
            if (b > 0) ludyn::c_to_b(make_double2(er0, ei0), make_double2(er1, ei1), lane, xb0[b], xb1[b]);
            const int row = kb + crow;
            if (ccol < 3) {
              Pw[ccol * R + row] = make_double2(er0, ei0);
              if (a.P_out && row < a.r)
                reinterpret_cast<double2 *>(a.P_out)[((size_t)t * 3 + ccol) * a.r + row] = make_double2(er0, ei0);
            }
            if (ccol + 1 < 3) {
              Pw[(ccol + 1) * R + row] = make_double2(er1, ei1);
              if (a.P_out && row < a.r)
                reinterpret_cast<double2 *>(a.P_out)[((size_t)t * 3 + ccol + 1) * a.r + row] = make_double2(er1, ei1);
            }
          }
        } else {
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
              ludyn::dmma(cr0, cr1, -a0.x, x0.x);
              ludyn::dmma(ci0, ci1, -a0.x, x0.y);
              ludyn::dmma(cr0, cr1, a0.y, x0.y);
              ludyn::dmma(ci0, ci1, -a0.y, x0.x);
              ludyn::dmma(cr0, cr1, -a1.x, x1.x);
              ludyn::dmma(ci0, ci1, -a1.x, x1.y);
              ludyn::dmma(cr0, cr1, a1.y, x1.y);
              ludyn::dmma(ci0, ci1, -a1.y, x1.x);
            } else {
              ludyn::dmma(dr0, dr1, -a0.x, x0.x);
              ludyn::dmma(di0, di1, -a0.x, x0.y);
              ludyn::dmma(dr0, dr1, a0.y, x0.y);
              ludyn::dmma(di0, di1, -a0.y, x0.x);
              ludyn::dmma(dr0, dr1, -a1.x, x1.x);
              ludyn::dmma(di0, di1, -a1.x, x1.y);
              ludyn::dmma(dr0, dr1, a1.y, x1.y);
              ludyn::dmma(di0, di1, -a1.y, x1.x);
            }
          }
          __syncwarp();
          A[(kb + crow) * LDA + R + ccol] = make_double2(cr0 + dr0, ci0 + di0);
          A[(kb + crow) * LDA + R + ccol + 1] = make_double2(cr1 + dr1, ci1 + di1);
          __syncwarp();
          // x_b = Dinv_b y_b (Dinv_b stored in place of U11)
          double2 v0, v1;
          {
            const int m = arow, k0 = acol, k1 = acol + 4;
            v0 = m <= k0 ? A[(kb + m) * LDA + kb + k0] : make_double2(0.0, 0.0);
            v1 = m <= k1 ? A[(kb + m) * LDA + kb + k1] : make_double2(0.0, 0.0);
          }
          const double2 x0 = A[(kb + bk) * LDA + R + bcol], x1 = A[(kb + 4 + bk) * LDA + R + bcol];
          double er0 = 0.0, er1 = 0.0, ei0 = 0.0, ei1 = 0.0;
          ludyn::dmma(er0, er1, v0.x, x0.x);
          ludyn::dmma(ei0, ei1, v0.x, x0.y);
          ludyn::dmma(er0, er1, -v0.y, x0.y);
          ludyn::dmma(ei0, ei1, v0.y, x0.x);
          ludyn::dmma(er0, er1, v1.x, x1.x);
          ludyn::dmma(ei0, ei1, v1.x, x1.y);
          ludyn::dmma(er0, er1, -v1.y, x1.y);
          ludyn::dmma(ei0, ei1, v1.y, x1.x);
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
        }  // !RG
      } else {
        for (int e = lane; e < 3 * R; e += 32) Pw[e] = make_double2(nanv, nanv);
        if (a.P_out)
          for (int e = lane; e < 3 * a.r; e += 32)
            reinterpret_cast<double2 *>(a.P_out)[(size_t)t * 3 * a.r + e] = make_double2(nanv, nanv);
      }
      if (a.info && lane == 0) a.info[t] = info;
    }
    if constexpr (W > 1) ludyn::bar_sync(bar_id, NT); else __syncwarp();
  }
}

template <int R, int W, bool RG>
static cudaError_t launch_lu_dyn_k(const EvalArgs &a, cudaStream_t s);

template <int R, int W>
static cudaError_t launch_lu_dyn_t(const EvalArgs &a, cudaStream_t s) {
  // RG (right-hand sides in L2) only where it buys a group per SM and the scratch exists
  constexpr bool RG = ludyn::Cfg<R, W, true>::GROUPS > ludyn::Cfg<R, W, false>::GROUPS;
  if constexpr (RG) {
    if (a.gscr) return launch_lu_dyn_k<R, W, true>(a, s);
  }
  return launch_lu_dyn_k<R, W, false>(a, s);
}

template <int R, int W, bool RG>
static cudaError_t launch_lu_dyn_k(const EvalArgs &a, cudaStream_t s) {
  using C = ludyn::Cfg<R, W, RG>;
  auto kern = lu_dyn_kernel<R, W, RG>;
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

// measured on B200 (tools/lu_ab.py, F = 1e5): one warp per frequency up to R = 40, two at R = 48, 56, 72 and 80,
// four at R = 64, 88 and 96.  The right-hand-side-in-L2 (RG) variant is instantiated only where it buys a group
// per SM (launch_lu_dyn_t): R = 48 (6 instead of 5) and R = 56 (4 instead of 3); at R = 80 both layouts fit 2
static int dyn_warps(int R) { return R <= 40 ? 1 : ((R == 48 || R == 56 || R == 72 || R == 80) ? 2 : 4); }

template <int R>
static bool dyn_uses_rg() {
  switch (dyn_warps(R)) {
    case 1: return ludyn::Cfg<R, 1, true>::GROUPS > ludyn::Cfg<R, 1, false>::GROUPS;
    case 2: return ludyn::Cfg<R, 2, true>::GROUPS > ludyn::Cfg<R, 2, false>::GROUPS;
    default: return ludyn::Cfg<R, 4, true>::GROUPS > ludyn::Cfg<R, 4, false>::GROUPS;
  }
}

// L2 scratch of the RG variant; 0 where the launch uses the shared-memory layout (no 16 MB allocation
// per evaluation for nothing)
size_t lu_dyn_scratch_bytes(int R, int sms) {
  bool rg = false;
  switch (R) {
#define PODP_CASE(RR) \
  case RR: rg = dyn_uses_rg<RR>(); break;
    PODP_CASE(8) PODP_CASE(16) PODP_CASE(24) PODP_CASE(32) PODP_CASE(40) PODP_CASE(48) PODP_CASE(56) PODP_CASE(64)
    PODP_CASE(72) PODP_CASE(80) PODP_CASE(88) PODP_CASE(96)
#undef PODP_CASE
    default: break;
  }
  return rg ? (size_t)sms * 16 * 9 * R * sizeof(double2) : 0;
}

cudaError_t launch_lu_dyn(const EvalArgs &a, cudaStream_t s) {
  if (a.flags & PODP_FLAG_NO_PIVOT) return cudaErrorNotSupported;
  const int R = a.L.R;
  const int wv = dyn_warps(R);
  switch (R) {
#define PODP_CASE(RR)                                     \
  case RR:                                                \
    if (wv == 1) return launch_lu_dyn_t<RR, 1>(a, s);     \
    if (wv == 2) return launch_lu_dyn_t<RR, 2>(a, s);     \
    return launch_lu_dyn_t<RR, 4>(a, s);
#ifdef PODP_DEV_R  // dev builds: a single instantiation
    case PODP_DEV_R: return launch_lu_dyn_t<PODP_DEV_R, PODP_DEV_W>(a, s);
#else
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
#endif
#undef PODP_CASE
    default: return cudaErrorNotSupported;
  }
}

}  // namespace podp
