// K2 default path (R <= 96): left-looking block LU with partial pivoting + 3-RHS solve, ONE WARP PER FREQUENCY
// (rows a2-a3 of SURVEY 8(a)).
//   A(omega) = K + i omega nu M,  B(omega) = b0 + omega b1,  P = A^{-1} B            (eqn:ReducedA)
//
// Factorisation (the same pivots and the same trailing updates as LAPACK's blocked getrf, reordered):
//   P_perm A = Lhat Uhat,  Lhat = [I; M_tb] block unit lower (8x8 identity diagonal blocks),
//   Uhat = [Y_tc (t < c); Uhat_cc = L_cc U_cc] block upper, where for 8-column panel c (rows 8c .. R-1, after the
//   updates of panels 0..c-1) P_c [A_cc; A_tc] = [L_cc; L_tc] U_cc is an unblocked LU with partial pivoting,
//   M_tc = L_tc L_cc^{-1}, and Y_tc = A_tc - sum_{b<t} M_tb Y_bc is block (t, c) of the right-looking getrf
//   update before its L_tt^{-1} solve (U_tc = L_tt^{-1} Y_tc).  Then z = Lhat^{-1} P_perm B (forward, 3 columns)
//   and x = Uhat^{-1} z (block back substitution with D_t = Uhat_tt^{-1}).
//
// Layout.  Column tile c (8 columns) is accumulated in REGISTERS as DMMA C fragments (acc_t, t = 0..NT-1):
//   acc = A[perm rows, c] - sum_b M_{:,b} Y_{b,c} on mma.sync.m8n8k4.f64 (SASS DMMA; a complex 8x8x8 tile product is
//   8 DMMA), so trailing-update results never round-trip through shared memory; only the M strips (M_{t,b}, read
//   as A fragments, XOR-swizzled rows: conflict-free both as A fragments and as lane = row panel rows) live in the
//   warp's shared-memory slice.  Y_{t,c} (t < c) and D_t go to a per-warp L2-resident scratch (read once by the
//   back substitution).  The panel is factored in registers with lane = row (redux.sync argmax of an integer
//   magnitude key, pivot-row broadcast through 9 complex of shared memory, speculative per-candidate reciprocals
//   so the reciprocal is off the pivot chain).  Rows never move: a position -> physical-row map (perm) gathers K
//   and M rows at assembly time and the M strips of earlier panels are re-ordered only when a panel interchanged
//   rows.  The 3-column right-hand side is real-ified (8 x [Re | Im] columns): a complex 8x8 by 8x3 product is 4 DMMA.
//   One warp owns one frequency end to end (no inter-warp synchronisation); G independent warps per CTA.
//   Shared memory per warp holds only the M tiles (NT(NT-1)/2) plus one tile for the current panel's diagonal block
//   (see strip_off): the diagonal blocks go to the L2 scratch with the Y tiles, which buys warps per SM (r = 48:
//   12 instead of 10, r = 96: 3 instead of 2; measured 3.47 -> 3.29 ms and 48.4 -> 33.1 ms per 1e5 frequencies).
//   Round-2 additions (each measured): M tiles in TENSOR MEMORY with K and M staged in shared
//   memory (Cfg::TM), strips beyond tensor memory in the L2 scratch (HYB_G), a CTA rendezvous every 16th frequency at
//   R = 48 so that the warps share the instruction cache (LOCKSTEP), Gauss's three-product complex multiplication in
//   the updates (GAUSS3), conflict-free strip swizzle and padded staging of the diagonal blocks, Y tiles converted
//   from C to B fragments through a free strip tile (body, stg).
#include <utility>

#include "podp_common.cuh"

// Dev-only phase ablation for throughput attribution (never defined in the product build): bit 0 skips the panel's
// arithmetic, 1 the left-looking updates, 2 the diagonal-block inverses, 3 the forward/back substitution; inside the
// panel: 4 the M = L L_cc^{-1} solve, 5 the rank-1 updates except of the next column, 6 the pivot reciprocals.
#ifndef PODP_LL_ABLATE
#define PODP_LL_ABLATE 0
#endif
// Dev: PODP_LL_SYNC = 0 / 1 forces the per-frequency CTA rendezvous (Cfg::LOCKSTEP) off / on for every size.
#ifndef PODP_LL_SROW_MAX
#define PODP_LL_SROW_MAX 40
#endif

namespace podp {

namespace lull {

template <int R, bool KM = false, bool TM = false>
struct Cfg {
  static_assert(R % 8 == 0 && R >= 8 && R <= 96, "left-looking kernel: R in 8..96, multiple of 8");
  static constexpr int NT = R / 8;                       // tile rows / columns
  // DIAG_L2 (R >= 40, where shared memory bounds the warps per SM): shared memory per warp holds the M tiles of
  // every strip (strip b: tiles b+1..NT-1) plus one tile for the diagonal block of the panel being factored (see
  // strip_off), and the diagonal blocks go to the L2 scratch; below, strip b holds tiles b..NT-1 including its
  // diagonal block (measured faster there: no copy-out, and the warp count is capped by registers anyway)
  static constexpr bool DIAG_L2 = R >= 40 || TM;
  // TM (single-object launches, 40 <= R <= 64): the M tiles live in TENSOR MEMORY (tcgen05.st / tcgen05.ld, one
  // 8-column slice per tile in A-fragment order, this warp's 32 TMEM lanes); shared memory keeps only the current
  // panel's virtual strip (NT tiles, also the scratch of the row interchanges and of the final inverses), so K and M
  // fit in shared memory beside 12 warps' state (KM)
  // strips 0 .. TM_TB-1 live in tensor memory (TM_COLS columns per warp, 512 / TM_COLS warps per SM sub-partition);
  // the remaining strips stay in shared memory after the virtual strip.  TM_COLS is chosen to maximise the warps per
  // SM under the shared-memory, register and tensor-memory limits (r = 48: all 15 tiles in 128 columns, 12 warps;
  // r = 80: 4 strips in 256 columns, 8 warps instead of 4; r = 96: 9 strips in 512 columns, 4 instead of 3)
  // HYB_G (R >= 88): the strips that do not fit in tensor memory go to the warp's L2 scratch instead of shared
  // memory, so that the warp count is set by tensor memory and registers (r = 96: 8 warps instead of 4)
  static constexpr bool HYB_G = TM && R >= 88;
  static constexpr int tm_tiles(int tb) { return tb * (NT - 1) - tb * (tb - 1) / 2; }
  static constexpr int tm_fit(int cols) {
    int tb = 0;
    while (tb < NT - 1 && 8 * tm_tiles(tb + 1) <= cols) ++tb;
    return tb;
  }
  static constexpr int PERM_BYTES = ((R * 4 + 15) / 16) * 16;
  #ifndef PODP_LL_GREG48
#define PODP_LL_GREG48 12
#endif
  static constexpr int G_REG = R <= 32 ? 16 : (R <= 40 ? 12 : (R <= 48 ? PODP_LL_GREG48 : 8));  // register cap, see below
  static constexpr int tm_warps(int cols) {
    const int hyb = NT * (NT - 1) / 2 - tm_tiles(tm_fit(cols));
    const int w_bytes = (NT + (HYB_G ? 0 : hyb)) * 1024 + 9 * 16 + 2 * PERM_BYTES;
    const int km = R <= 64 ? 2 * R * (R + 1) * 16 : 0;
    const int g_smem = (227 * 1024 - km) / w_bytes, g_tm = 4 * (512 / cols);
    const int g = g_smem < G_REG ? g_smem : G_REG;
    return g < g_tm ? g : g_tm;
  }
  static constexpr int tm_best_cols() {
    int best = 512;
    for (int cols = 256; cols >= 64; cols /= 2)
      if (tm_warps(cols) > tm_warps(best)) best = cols;
    return best;
  }
  static constexpr int TM_COLS = TM ? tm_best_cols() : 64;
  static constexpr int TM_TB = TM ? tm_fit(TM_COLS) : 0;
  static constexpr int TM_TILES = tm_tiles(TM_TB);       // M tiles per frequency in TMEM (8 columns each)
  static constexpr int HYB_TILES = NT * (NT - 1) / 2 - TM_TILES;
  static constexpr int STRIP_TILES =
      TM ? NT + (HYB_G ? 0 : HYB_TILES) : (DIAG_L2 ? 1 + NT * (NT - 1) / 2 : NT * (NT + 1) / 2);
  static constexpr int MS = (R + 31) / 32;               // panel row slots per lane
  // staging tile for the right-hand-side fragment conversions (rhs_frags through shared memory instead of shuffles):
  // dev option, off -- fewer instructions but a longer back-substitution chain, r = 48: 2.518 vs 2.512 ms
#ifdef PODP_LL_ZT
  static constexpr int ZT_BYTES = TM ? 512 : 0;
#else
  static constexpr int ZT_BYTES = 0;
#endif
  static constexpr int W_BYTES = STRIP_TILES * 1024 + 9 * 16 + ((R * 4 + 15) / 16) * 16 * (TM ? 2 : 1) + ZT_BYTES;
  // KM (single-object launches, R <= 40, or with TM): K and M staged once per CTA in shared memory (row stride
  // R + 1 complex), so the column-tile gathers are shared-memory loads instead of L2 round trips (r = 40: 2.27 ->
  // 2.10 ms per 1e5 at the same 12 warps; without TM, at R >= 48 the copy would cost warps, measured slower)
  // (+ b0 and b1, 3R complex each, read by the right-hand-side assembly of every frequency)
  static constexpr int KM_BYTES = (KM || TM) && R <= 64 ? (2 * R * (R + 1) + 6 * (R + 2)) * 16 : 0;
  static constexpr int G_SMEM = (227 * 1024 - KM_BYTES) / W_BYTES;
  // warp cap G_REG (measured: ptxas allocates <= 168 registers up to R = 48, i.e. 3 warps per SM sub-partition,
  // 224-255 above, i.e. 2; at R <= 32 16 warps with 128 registers are fastest)
#ifdef PODP_LL_G  // dev: fewer warps per CTA (occupancy experiments)
  static constexpr int G_MAX = R <= 48 ? PODP_LL_G : G_REG;
#else
  static constexpr int G_MAX = G_REG;
#endif
  static constexpr int G_TM = TM ? 4 * (512 / TM_COLS) : 64;
  static constexpr int G_SR = G_SMEM < G_MAX ? G_SMEM : G_MAX;
  static constexpr int G = G_SR < G_TM ? G_SR : G_TM;    // warps (= concurrent frequencies) per CTA
  static_assert(!TM || TM_COLS * ((G + 3) / 4) <= 512, "M tiles do not fit in tensor memory");
  // per-warp L2 scratch: Y_{t,c} (t < c): NT(NT-1)/2, D_t: NT, L\U diag: NT (+ HYB_G: the hybrid strips)
  // LOCKSTEP: the warps of a CTA start every frequency together (one __syncthreads per frequency).  The kernel is
  // ~150 KB of straight-line code that each warp streams once per frequency; 12 warps at 12 different places miss the
  // SM's instruction cache (ncu at r = 48: icc hit rate 86 %, GPC-level instruction requests at 67 % of peak,
  // no_instruction 0.72 stall cycles per issue); in step they share each fetched line (hit rate 96 %, requests 26 %):
  // r = 48 solve 3.13 -> 2.84 ms per 1e5.  Measured slower where the code is smaller or fewer warps run (R <= 40:
  // 0.5-8 %; R >= 56: 0-1.5 %), so only the R = 48 tensor-memory variant takes it.
  // GAUSS3: three-product complex tile multiplication in the left-looking updates (see body): 330 instead of 440
  // DMMA per frequency at r = 48.  Measured per 1e5: r = 40 2.07 -> 1.95 ms, r = 48 2.76 -> 2.68, r = 64 5.45 -> 5.38,
  // r = 32 1.18 -> 1.17, r = 72 8.08 -> 8.02, r = 80 10.31 -> 10.09; not faster at r <= 24 (few updates) and slower at
  // r = 88 (16.39 vs 16.16) and r = 96 (20.1 vs 19.7): registers
#ifdef PODP_LL_GAUSS3
  static constexpr bool GAUSS3 = PODP_LL_GAUSS3 != 0;
#else
  static constexpr bool GAUSS3 = R >= 32 && R <= 80;
#endif
#ifdef PODP_LL_SYNC
  static constexpr bool LOCKSTEP = PODP_LL_SYNC != 0;
#else
  static constexpr bool LOCKSTEP = TM && R == 48;
#endif
  // the rendezvous is taken every LOCKSTEP_EVERY-th frequency (power of two): the warps drift apart slowly, and a
  // barrier per frequency costs its wait for the slowest warp (r = 48: every 1 / 4 / 16 / 64: 2.65 / 2.60 / 2.58 /
  // 2.59 ms per 1e5)
#ifdef PODP_LL_SYNC_EVERY
  static constexpr int LOCKSTEP_EVERY = PODP_LL_SYNC_EVERY;
#else
  static constexpr int LOCKSTEP_EVERY = 16;
#endif
  static constexpr int GSCR_TILES = NT * (NT + 3) / 2 + (HYB_G ? HYB_TILES : 0);
  static constexpr size_t BYTES = (size_t)G * W_BYTES + KM_BYTES;
  static_assert(G >= 1, "strips do not fit in shared memory");
  static_assert(TM || !DIAG_L2 || 2 * NT * 65 <= STRIP_TILES * 64 + 9,
                "diagonal blocks and D_t (stride 65) must fit in the strip area");
};

// Shared-memory tile offset of the "virtual strip" of panel b: its diagonal-block tile followed by its M tiles
// (tiles b+1..NT-1).  Without DIAG_L2 the strips are simply consecutive (strip b = tiles b..NT-1).  With DIAG_L2 the
// strips are stored in reverse order after one spare tile, [spare | strip NT-2 | strip NT-3 | ... | strip 0] (M tiles
// only), so the diagonal-block tile of panel b is the last tile of strip b+1 (or the spare tile): space that is
// written only after panel b has copied its diagonal block to the L2 scratch.  Every access to the M tiles of strip
// b is at tile offset >= 1 from strip_off(b), in both layouts.
// TM, strips b >= TB kept in shared memory (R = 96): strip b's virtual base sits so that its tile t is at tile
// NT + (tiles of strips TB .. b-1) + (t - b - 1), i.e. base = NT - 1 + sum_{TB <= b' < b} (NT - 1 - b')
__host__ __device__ constexpr int strip_off_hyb(int NT, int TB, int b) {
  return NT - 1 + (b - TB) * (NT - 1) - (b * (b - 1) - TB * (TB - 1)) / 2;
}
template <bool DIAG_L2>
__host__ __device__ constexpr int strip_off(int NT, int b) {
  return DIAG_L2 ? (NT - 2 - b) * (NT - 1 - b) / 2 : b * NT - b * (b - 1) / 2;
}
// row swizzle: slot = k ^ swz(i & 7) makes lane = row accesses (8 rows, same k), A-fragment reads (rows 2j, 2j+1 x
// 4 consecutive k: the two rows' swizzles differ in bit 2) and C-fragment stores (rows 2j, 2j+1 x even or odd k: they
// differ in bit 0) each hit 8 distinct 16-byte bank groups
__device__ __forceinline__ int swz(int i) { return ((i & 1) * 5) ^ ((i >> 1) & 3); }

__device__ __forceinline__ double selp_f64(double a, double b, int p) {  // p ? a : b
  double r;
  asm("{\n .reg .pred q;\n setp.ne.s32 q, %3, 0;\n selp.f64 %0, %1, %2, q;\n}" : "=d"(r) : "d"(a), "d"(b), "r"(p));
  return r;
}
__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// ---- tensor memory (tcgen05) helpers: 32x32b shape, thread i <-> TMEM lane (32 * (warp % 4) + i) ---------------
__device__ __forceinline__ void tm_st8(uint32_t taddr, double2 m0, double2 m1) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
               "r"(__double2loint(m0.x)), "r"(__double2hiint(m0.x)), "r"(__double2loint(m0.y)), "r"(__double2hiint(m0.y)),
               "r"(__double2loint(m1.x)), "r"(__double2hiint(m1.x)), "r"(__double2loint(m1.y)), "r"(__double2hiint(m1.y))
               : "memory");
}
__device__ __forceinline__ void tm_ld8(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr)
               : "memory");
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ double2 tm_m0(const uint32_t (&v)[8]) {
  return make_double2(__hiloint2double(v[1], v[0]), __hiloint2double(v[3], v[2]));
}
__device__ __forceinline__ double2 tm_m1(const uint32_t (&v)[8]) {
  return make_double2(__hiloint2double(v[5], v[4]), __hiloint2double(v[7], v[6]));
}
// TMEM column of M tile (strip b, tile t > b) of one frequency: strip b holds NT - 1 - b tiles
__host__ __device__ constexpr int tm_tile(int NT, int b, int t) { return b * (NT - 1) - b * (b - 1) / 2 + (t - b - 1); }

// B fragment (k = 4s + lane%4, n = lane/4) of an 8x8 tile held as C fragments (row lane/4, cols 2(lane%4) + {0,1})
__device__ __forceinline__ double frag_c2b(double c0, double c1, int s, int lane) {
  const int src = 16 * s + 4 * (lane & 3) + (lane >> 3);
  const double v0 = __shfl_sync(0xffffffffu, c0, src), v1 = __shfl_sync(0xffffffffu, c1, src);
  return ((lane >> 2) & 1) ? v1 : v0;
}

// Real-ified right-hand side tile Z = [Re z_0..2 | Im z_0..2 | 0 0] (C fragments) -> B fragments of Z (b1) and of
// Z' = [-Im z | Re z | 0 0] (b2), so that a complex 8x8 A times z is  Re(A) Z + Im(A) Z'  (2 DMMA per k-step).
// zt != nullptr (tensor-memory variants): through a 512-byte row-major staging tile in shared memory (1 store + 4 loads
// instead of 16 shuffles and their selects).
__device__ __forceinline__ void rhs_frags(double c0, double c1, int lane, double (&b1)[2], double (&b2)[2],
                                          double *zt = nullptr) {
  const int n = lane >> 2;
  const int j2 = n < 3 ? n + 3 : (n < 6 ? n - 3 : 6);
  if (zt) {
    __syncwarp();  // earlier loads from the tile are done
    reinterpret_cast<double2 *>(zt)[lane] = make_double2(c0, c1);  // Z[lane / 4][2 (lane % 4) + {0, 1}]
    __syncwarp();
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int k = 4 * s + (lane & 3);
      b1[s] = zt[k * 8 + n];
      const double w = zt[k * 8 + j2];
      b2[s] = n < 3 ? -w : (n < 6 ? w : 0.0);
    }
    return;
  }
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int row = 4 * (4 * s + (lane & 3));
    const int src1 = row + (n >> 1), src2 = row + (j2 >> 1);
    const double u0 = __shfl_sync(0xffffffffu, c0, src1), u1 = __shfl_sync(0xffffffffu, c1, src1);
    const double w0 = __shfl_sync(0xffffffffu, c0, src2), w1 = __shfl_sync(0xffffffffu, c1, src2);
    b1[s] = (n & 1) ? u1 : u0;
    const double w = (j2 & 1) ? w1 : w0;
    b2[s] = n < 3 ? -w : (n < 6 ? w : 0.0);
  }
}

// Column c, block b: Y_{b,c} = acc_b is final -> scratch (C-fragment order) and acc_t -= M_{t,b} Y_{b,c}, t > b.
// The M tiles come from shared memory, or (TM) from tensor memory: one tcgen05.ld per tile, one wait for all.
// M3 (Gauss's three-product complex multiplication): with Ms = Mr + Mi, the three running sums
//   ak -= Ms Yr,  ar += Mi (Yr + Yi),  ai += Mr (Yr - Yi)   give   Re = ar + ak,  Im = ai + ak
// (Re(MY) = Ms Yr - Mi (Yr + Yi), Im(MY) = Ms Yr + Mr (Yi - Yr)): 6 DMMA per complex tile product instead of 8, for
// one more accumulator set per column tile and 2 additions per M tile; ar/ai of tile B are final only as ar + ak,
// ai + ak (formed here for Y_{B,c}, and by column_tile for the rows that go to the panel).
// STG (tensor-memory variants): Y_{B,c} goes from C fragments to B fragments through one tile of the free
// virtual strip (2 stores + 2 loads, XOR mask 2 (row & 3) | (row & 1): conflict-free both ways) instead of 16 shuffles
// and 8 selects.
template <int NT, int B, bool TM = false, bool M3 = false>
__device__ __forceinline__ void body(double (&ar)[NT][2], double (&ai)[NT][2], double (&ak)[NT][2], const double2 *S,
                                     double2 *gY, int lane, uint32_t tm = 0, double2 *stg = nullptr) {
  if constexpr (M3) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      ar[B][e] += ak[B][e];
      ai[B][e] += ak[B][e];
    }
  }
  gY[2 * lane] = make_double2(ar[B][0], ai[B][0]);
  gY[2 * lane + 1] = make_double2(ar[B][1], ai[B][1]);
  double nyr[2], yi[2], nyi[2];  // M3: -Yr, Yr + Yi, Yr - Yi
  const int r4 = lane >> 2, q = lane & 3;
#ifndef PODP_LL_NO_STG
  constexpr bool STG = TM;
#else
  constexpr bool STG = false;
#endif
  if constexpr (STG) {
    const int fw = ((r4 & 3) << 1) | (r4 & 1);
    __syncwarp();  // the previous block's loads from the staging tile are done
    stg[r4 * 8 + ((2 * q) ^ fw)] = make_double2(ar[B][0], ai[B][0]);
    stg[r4 * 8 + ((2 * q + 1) ^ fw)] = make_double2(ar[B][1], ai[B][1]);
    __syncwarp();
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int k = 4 * s + q;  // B fragment: Y[k][n = r4]
      const double2 y = stg[k * 8 + (r4 ^ (((k & 3) << 1) | (k & 1)))];
      nyr[s] = -y.x;
      yi[s] = M3 ? y.x + y.y : y.y;
      nyi[s] = M3 ? y.x - y.y : -y.y;
    }
  } else {
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const double r = frag_c2b(ar[B][0], ar[B][1], s, lane), i = frag_c2b(ai[B][0], ai[B][1], s, lane);
      nyr[s] = -r;
      yi[s] = M3 ? r + i : i;
      nyi[s] = M3 ? r - i : -i;
    }
  }
  constexpr int TB = Cfg<8 * NT, false, TM>::TM_TB;
  constexpr bool IN_TM = TM && B < TB;  // this strip in tensor memory (else shared memory)
  // TMEM loads in chunks of TMC tiles (one wait per chunk) to bound the registers they occupy
  constexpr int TMC = NT <= 9 ? 2 : 4;  // measured: 2 is ~1 % faster up to R = 72, 4 above (fewer waits)
  uint32_t v[NT][8];
  const double2 *Sb = S + (TM ? strip_off_hyb(NT, TB, B) : strip_off<Cfg<8 * NT>::DIAG_L2>(NT, B)) * 64;
  const int k0 = q ^ swz(r4), k1 = (4 + q) ^ swz(r4);
#pragma unroll
  for (int t = B + 1; t < NT; ++t) {
    if constexpr (IN_TM) {
      if ((t - B - 1) % TMC == 0) {
#pragma unroll
        for (int u = t; u < NT && u < t + TMC; ++u) tm_ld8(tm + 8 * tm_tile(NT, B, u), v[u]);
        tm_wait_ld();
      }
    }
    double2 m0, m1;
    if constexpr (IN_TM) {
      m0 = tm_m0(v[t]);
      m1 = tm_m1(v[t]);
    } else {
      const double2 *row = Sb + (8 * (t - B) + r4) * 8;
      m0 = row[k0];
      m1 = row[k1];
    }
    if constexpr (M3) {
      const double s0 = m0.x + m0.y, s1 = m1.x + m1.y;
      dmma(ak[t][0], ak[t][1], s0, nyr[0]);
      dmma(ar[t][0], ar[t][1], m0.y, yi[0]);
      dmma(ai[t][0], ai[t][1], m0.x, nyi[0]);
      dmma(ak[t][0], ak[t][1], s1, nyr[1]);
      dmma(ar[t][0], ar[t][1], m1.y, yi[1]);
      dmma(ai[t][0], ai[t][1], m1.x, nyi[1]);
    } else {
      // acc -= M Y :  Re += Mr (-Yr) + Mi Yi ;  Im += Mr (-Yi) + Mi (-Yr)
      dmma(ar[t][0], ar[t][1], m0.x, nyr[0]);
      dmma(ai[t][0], ai[t][1], m0.x, nyi[0]);
      dmma(ar[t][0], ar[t][1], m0.y, yi[0]);
      dmma(ai[t][0], ai[t][1], m0.y, nyr[0]);
      dmma(ar[t][0], ar[t][1], m1.x, nyr[1]);
      dmma(ai[t][0], ai[t][1], m1.x, nyi[1]);
      dmma(ar[t][0], ar[t][1], m1.y, yi[1]);
      dmma(ai[t][0], ai[t][1], m1.y, nyr[1]);
    }
  }
}

template <int NT, bool TM = false, bool M3 = false, int B = 0>
__device__ __forceinline__ void body_dispatch(int b, double (&ar)[NT][2], double (&ai)[NT][2], double (&ak)[NT][2],
                                              const double2 *S, double2 *gY, int lane, uint32_t tm = 0,
                                              double2 *stg = nullptr) {
  if constexpr (B < NT - 1) {
    if (b == B) body<NT, B, TM, M3>(ar, ai, ak, S, gY, lane, tm, stg);
    else body_dispatch<NT, TM, M3, B + 1>(b, ar, ai, ak, S, gY, lane, tm, stg);
  }
}

// Forward substitution z_t -= M_{t,B} z_B (real-ified right-hand side), t > B
template <int NT, int B, bool TM = false>
__device__ __forceinline__ void body_rhs(double (&z)[NT][2], const double2 *S, int lane, uint32_t tm = 0,
                                         double *zt = nullptr) {
  double b1[2], b2[2];
  rhs_frags(z[B][0], z[B][1], lane, b1, b2, zt);
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    b1[s] = -b1[s];
    b2[s] = -b2[s];
  }
  const int r4 = lane >> 2, q = lane & 3;
  constexpr int TB = Cfg<8 * NT, false, TM>::TM_TB;
  constexpr bool IN_TM = TM && B < TB;  // this strip in tensor memory (else shared memory)
  // TMEM loads in chunks of TMC tiles (one wait per chunk) to bound the registers they occupy
  constexpr int TMC = NT <= 9 ? 2 : 4;
  uint32_t v[NT][8];
  const double2 *Sb = S + (TM ? strip_off_hyb(NT, TB, B) : strip_off<Cfg<8 * NT>::DIAG_L2>(NT, B)) * 64;
  const int k0 = q ^ swz(r4), k1 = (4 + q) ^ swz(r4);
#pragma unroll
  for (int t = B + 1; t < NT; ++t) {
    if constexpr (IN_TM) {
      if ((t - B - 1) % TMC == 0) {
#pragma unroll
        for (int u = t; u < NT && u < t + TMC; ++u) tm_ld8(tm + 8 * tm_tile(NT, B, u), v[u]);
        tm_wait_ld();
      }
    }
    double2 m0, m1;
    if constexpr (IN_TM) {
      m0 = tm_m0(v[t]);
      m1 = tm_m1(v[t]);
    } else {
      const double2 *row = Sb + (8 * (t - B) + r4) * 8;
      m0 = row[k0];
      m1 = row[k1];
    }
    dmma(z[t][0], z[t][1], m0.x, b1[0]);
    dmma(z[t][0], z[t][1], m0.y, b2[0]);
    dmma(z[t][0], z[t][1], m1.x, b1[1]);
    dmma(z[t][0], z[t][1], m1.y, b2[1]);
  }
}

// A fragment (row lane/4, k = 4s + lane%4) of a complex tile stored in C-fragment order (element (i, k) at
// 2 * (4 i + k / 2) + k % 2), from the L2 scratch
__device__ __forceinline__ double2 afrag_cstore(const double2 *g, int s, int lane) {
  const int k = 4 * s + (lane & 3);
  return __ldcg(g + 2 * (4 * (lane >> 2) + (k >> 1)) + (k & 1));
}
// the same from shared memory, rows XOR-swizzled (element (i, k) at 8 i + (k ^ 4 (i & 1))): rows 2j and 2j+1 of a
// quarter warp fall into different halves of the 128-byte line pair (conflict-free)
__device__ __forceinline__ double2 afrag_cstore_s(const double2 *g, int s, int lane) {
  const int k = 4 * s + (lane & 3), i = lane >> 2;
  return g[8 * i + (k ^ ((i & 1) << 2))];
}

// Unblocked LU with partial pivoting of panel c (rows 8c .. R-1 of strip c, lane = row), M_tc = L_tc L_cc^{-1},
// interchanges applied to perm and to the strips of earlier panels.  Returns 0 or (LAPACK getrf info) k + 1 for
// an exactly zero pivot column at global step k.
template <int R, int MSE, bool PIVOT, bool TM = false>
__device__ __forceinline__ int panel(int c, double2 *S, double2 *sRow, int *sPerm, double2 *gDiag, int lane,
                                     uint32_t tm = 0, int *sMap = nullptr, double2 *Sh = nullptr) {
  constexpr int NT = R / 8;
  const int kb = 8 * c;
  double2 *St = TM ? S : S + strip_off<Cfg<8 * NT>::DIAG_L2>(NT, c) * 64;
  double2 pn[MSE][8], urc[MSE];
  int pos[MSE], q0[MSE], pv[MSE];
  bool alive[MSE];  // not yet chosen as a pivot row (and a real row)
  int bad = 0;       // LAPACK info of the first exactly zero pivot column
#pragma unroll
  for (int m = 0; m < MSE; ++m) {
    const int i = kb + lane + 32 * m;
    const bool v = i < R;
    q0[m] = i;
    pos[m] = v ? i : (1 << 20);
    pv[m] = v ? sPerm[i] : 0;
    alive[m] = v;
#pragma unroll
    for (int k = 0; k < 8; ++k) pn[m][k] = v ? St[(i - kb) * 8 + (k ^ swz(i & 7))] : make_double2(0.0, 0.0);
  }
  // Column step j.  Rows never move between lanes.  R >= 48: strip row h = slot (lane + 32 m) of the panel holds
  // that slot's current values, rewritten by its lane before each step (at j = 0 the strip already holds them), so
  // the pivot row is read straight from the strip once the argmax is known; its reciprocal (computed speculatively
  // by every candidate) and its position come by shuffle from the owning lane; the argmax key carries the slot
  // (ties: lowest slot).  R <= 40 (SROW): the pivot row's owner copies it to the 9-entry sRow and the key carries
  // the position (ties: lowest position) -- fewer shared-memory wavefronts, measured faster where 16 warps share
  // them (r = 24 .. 40: 1.5-3 %; R >= 48 the other way round, r = 64: 3 %).
  constexpr bool SROW = R <= PODP_LL_SROW_MAX;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int kr = kb + j;
    if (!SROW && j > 0) {
#pragma unroll
      for (int m = 0; m < MSE; ++m)
        if (alive[m]) {
          const int h = lane + 32 * m;
#pragma unroll
          for (int k = j + 1; k < 8; ++k) St[h * 8 + (k ^ swz(h & 7))] = pn[m][k];
        }
    }
    unsigned key = 0u;
    double2 rcm[MSE];
#pragma unroll
    for (int m = 0; m < MSE; ++m) {
      const unsigned tie = SROW ? (unsigned)(127 - (pos[m] & 127)) : (unsigned)(127 - lane - 32 * m);
      const unsigned kk = (mag_key_hi(pn[m][j]) & 0xFFFFFF80u) | tie;
      // candidates: every remaining row (partial pivoting) or only the row at position kr (PODP_FLAG_NO_PIVOT)
      if ((PIVOT ? alive[m] : pos[m] == kr) && kk > key) key = kk;
      if constexpr (PODP_LL_ABLATE & 64) rcm[m] = make_double2(1.0, 0.0);
      else rcm[m] = crecip_fast(pn[m][j]);  // speculative: off the chain after the argmax
    }
    if constexpr (!SROW) __syncwarp();  // the strip rows written above are visible to the warp
    const unsigned best = __reduce_max_sync(0xffffffffu, key);
    // exactly zero pivot column: return at once, or (48 <= R <= 64, measured 0.5-0.8 % faster there and 1-2 % slower
    // elsewhere) remember the first one and carry on without the branch -- the pivot is still a live row, so every
    // index stays valid, and the caller discards the frequency's results
    if constexpr (R <= 40 || R >= 72) {
      if ((best >> 7) == 0u) return kr + 1;
    } else {
      bad = (bad == 0 && (best >> 7) == 0u) ? kr + 1 : bad;
    }
    double2 rc, u[8];
    int p;
    bool piv[MSE];
    if constexpr (SROW) {
      p = 127 - (int)(best & 127u);
#pragma unroll
      for (int m = 0; m < MSE; ++m) {
        piv[m] = pos[m] == p;
        if (piv[m]) {
          const double d = fma(pn[m][j].x, pn[m][j].x, pn[m][j].y * pn[m][j].y);
          sRow[8] = (d >= 1e-290 && d <= 1e290) ? rcm[m] : crecip_scaled(pn[m][j]);  // call-free slow path
#pragma unroll
          for (int k = j + 1; k < 8; ++k) sRow[k] = pn[m][k];
        }
      }
      __syncwarp();
      rc = sRow[8];
#pragma unroll
      for (int k = j + 1; k < 8; ++k) u[k] = sRow[k];
    } else {
      const int ph = min(127 - (int)(best & 127u), 32 * MSE - 1), pl = ph & 31;
      // pivot reciprocal: crecip_fast is exact to ~1 ulp while max(|Re|,|Im|) is in [2^-480, 2^478) (|z|^2
      // normal); outside (warp-uniform, decided from the key's exponent bits) it is recomputed with crecip_scaled
      if (const unsigned bh = best & 0xFFFFFF80u; bh < 0x21F00000u || bh >= 0x5DD00000u) {
#pragma unroll
        for (int m = 0; m < MSE; ++m) rcm[m] = crecip_scaled(pn[m][j]);  // call-free slow path
      }
      double2 rsrc = rcm[0];
      int psrc = pos[0];
#pragma unroll
      for (int m = 1; m < MSE; ++m) {  // opaque selects: never an indexed local array
        const int sel = (ph >> 5) == m;
        rsrc = make_double2(selp_f64(rcm[m].x, rsrc.x, sel), selp_f64(rcm[m].y, rsrc.y, sel));
        psrc = sel ? pos[m] : psrc;
      }
      rc = make_double2(__shfl_sync(0xffffffffu, rsrc.x, pl), __shfl_sync(0xffffffffu, rsrc.y, pl));
      p = __shfl_sync(0xffffffffu, psrc, pl);
#pragma unroll
      for (int k = j + 1; k < 8; ++k) u[k] = St[ph * 8 + (k ^ swz(ph & 7))];
#pragma unroll
      for (int m = 0; m < MSE; ++m) piv[m] = lane + 32 * m == ph;
    }
#pragma unroll
    for (int m = 0; m < MSE; ++m) {
      pos[m] = piv[m] ? kr : (pos[m] == kr ? p : pos[m]);
      if (piv[m]) urc[m] = rc;  // 1/U_kk, kept for the diagonal-block inverse
      alive[m] = alive[m] && !piv[m];
    }
#pragma unroll
    for (int m = 0; m < MSE; ++m) {
      const bool act = alive[m];
      const double2 l = act ? cmul(pn[m][j], rc) : make_double2(0.0, 0.0);
      if (act) pn[m][j] = l;
#pragma unroll
      for (int k = j + 1; k < 8; ++k)
        if (!(PODP_LL_ABLATE & 32) || k == j + 1) pn[m][k] = cfms(l, u[k], pn[m][k]);
    }
    if constexpr (SROW) __syncwarp();  // sRow is rewritten by the next column
  }
  __syncwarp();  // every lane has read its last pivot row before the strip is rewritten below
  // diagonal block L_cc \ U_cc -> strip c rows 0..7, with 1/U_kk stored in place of U_kk (the diagonal entries
  // are used only by the diagonal-block inverse D_c, which needs the reciprocals)
#pragma unroll
  for (int m = 0; m < MSE; ++m)
    if (pos[m] >= kb && pos[m] < kb + 8) {
      double2 *rowp = St + (pos[m] - kb) * 8;
      const int sw = swz(pos[m] & 7);
#pragma unroll
      for (int k = 0; k < 8; ++k) rowp[k ^ sw] = pn[m][k];
      rowp[(pos[m] - kb) ^ sw] = urc[m];  // same lane, program order: the reciprocal replaces U_kk
    }
  __syncwarp();
  // rows below: m L_cc = l  (k = 7 .. 0: m_k = l_k - sum_{jj > k} m_jj L_cc[jj][k]), then store M rows
  if (kb + 8 < R) {
#pragma unroll
    for (int k = 6; k >= 0; --k) {
#pragma unroll
      for (int jj = 7; jj > k; --jj) {  // descending: the freshest m_jj enters each dependent chain last
        const double2 L = St[jj * 8 + (k ^ swz(jj))];
#pragma unroll
        for (int m = 0; m < MSE; ++m)
          if constexpr (!(PODP_LL_ABLATE & 16)) pn[m][k] = cfms(pn[m][jj], L, pn[m][k]);
      }
    }
#pragma unroll
    for (int m = 0; m < MSE; ++m)
      if (pos[m] >= kb + 8 && pos[m] < R) {
#pragma unroll
        for (int k = 0; k < 8; ++k) St[(pos[m] - kb) * 8 + (k ^ swz(pos[m] & 7))] = pn[m][k];
      }
  }
  if constexpr (TM) {
    // diagonal block -> L2 scratch; the panel's M tiles (rows of tiles c+1..NT-1) -> tensor memory in A-fragment
    // order (lane (r4, q) keeps M[r4][q] and M[r4][q + 4] of each tile); the shared-memory strip is then free
    __syncwarp();
    gDiag[c * 64 + lane] = St[lane];
    gDiag[c * 64 + 32 + lane] = St[32 + lane];
    const int r4 = lane >> 2, q = lane & 3;
    constexpr int TB = Cfg<R, false, TM>::TM_TB;
    if (c < TB) {
#pragma unroll
      for (int t = 1; t < NT; ++t)
        if (t > c) {
          const double2 *row = St + (8 * (t - c) + r4) * 8;
          tm_st8(tm + 8 * tm_tile(NT, c, t), row[q ^ swz(r4)], row[(4 + q) ^ swz(r4)]);
        }
      tm_wait_st();
    } else {  // (R >= 72) strips TB.. stay in shared memory after the virtual strip (HYB_G: in the L2 scratch)
      double2 *dst = Sh + strip_off_hyb(NT, TB, c) * 64;
      for (int e = 64 + lane; e < (NT - c) * 64; e += 32) dst[e] = St[e];
    }
    __syncwarp();
  }
  // interchanges: perm and the rows [kb, R) of the strips of earlier panels follow the panel's row movement
  bool moved = false;
#pragma unroll
  for (int m = 0; m < MSE; ++m) moved |= (pos[m] < R && pos[m] != q0[m]);
  if (__any_sync(0xffffffffu, moved)) {
#pragma unroll
    for (int m = 0; m < MSE; ++m)
      if (pos[m] < R && pos[m] != q0[m]) sPerm[pos[m]] = pv[m];
    // shared-memory strips: swap the moved rows in place (row i of strip b at Sb + 8 i)
    auto swap_rows_smem = [&](double2 *Sb) {
#pragma unroll
      for (int h = 0; h < 8; h += 4) {  // 4 columns at a time: all reads of a column precede its writes
        double2 tmp[MSE][4];
#pragma unroll
        for (int m = 0; m < MSE; ++m)
          if (pos[m] < R && pos[m] != q0[m]) {
#pragma unroll
            for (int k = 0; k < 4; ++k) tmp[m][k] = Sb[q0[m] * 8 + ((h + k) ^ swz(q0[m] & 7))];
          }
        __syncwarp();
#pragma unroll
        for (int m = 0; m < MSE; ++m)
          if (pos[m] < R && pos[m] != q0[m]) {
#pragma unroll
            for (int k = 0; k < 4; ++k) Sb[pos[m] * 8 + ((h + k) ^ swz(pos[m] & 7))] = tmp[m][k];
          }
        __syncwarp();
      }
    };
    if constexpr (TM) {
      // row p (>= kb) of every earlier strip takes the old row sMap[p]: tiles c..NT-1 of strip b are read from
      // tensor memory, laid out row-major in the (free) shared-memory strip, and written back permuted
      constexpr int TB = Cfg<R, false, TM>::TM_TB;
      const int r4 = lane >> 2, q = lane & 3;
      for (int p = kb + lane; p < R; p += 32) sMap[p] = p;
      __syncwarp();
#pragma unroll
      for (int m = 0; m < MSE; ++m)
        if (pos[m] < R && pos[m] != q0[m]) sMap[pos[m]] = q0[m];
      __syncwarp();
      for (int b = 0; b < c; ++b) {
        if (b >= TB) {
          swap_rows_smem(Sh + strip_off_hyb(NT, TB, b) * 64 - 8 * 8 * b);
          continue;
        }
#pragma unroll 1
        for (int t = c; t < NT; ++t) {  // one tile at a time (registers)
          uint32_t v[8];
          tm_ld8(tm + 8 * tm_tile(NT, b, t), v);
          tm_wait_ld();
          double2 *row = St + (8 * (t - c) + r4) * 8;
          row[q] = tm_m0(v);
          row[4 + q] = tm_m1(v);
        }
        __syncwarp();
#pragma unroll 1
        for (int t = c; t < NT; ++t) {
          const double2 *src = St + (sMap[8 * t + r4] - kb) * 8;
          tm_st8(tm + 8 * tm_tile(NT, b, t), src[q], src[4 + q]);
        }
        tm_wait_st();
        __syncwarp();
      }
    } else {
      for (int b = 0; b < c; ++b) swap_rows_smem(S + strip_off<Cfg<8 * NT>::DIAG_L2>(NT, b) * 64 - 8 * 8 * b);
    }
  }
  __syncwarp();
  if constexpr (Cfg<R>::DIAG_L2 && !TM) {
    // the diagonal block (L_cc \ U_cc with 1/U_kk on the diagonal, swizzled rows) -> L2 scratch for the inverses;
    // its shared-memory tile is reused by the next strip
    gDiag[c * 64 + lane] = St[lane];
    gDiag[c * 64 + 32 + lane] = St[32 + lane];
    __syncwarp();
  }
  return bad;
}

}  // namespace lull

namespace lull {

// a2 + the left-looking updates of column tile c for one frequency: A[perm rows, c] = K + i s M gathered into C
// fragments, minus sum_{b < c} M_{:,b} Y_{b,c} (DMMA), then rows >= 8c to the panel's virtual strip.
template <int R, bool TM = false>
__device__ __forceinline__ void column_tile(int c, double (&ar)[R / 8][2], double (&ai)[R / 8][2], double2 *S,
                                            double2 *gY, const int *sPerm, const double2 *gK, const double2 *gM,
                                            double s, int lane, int ldkm = R, uint32_t tm = 0,
                                            const double2 *Sh = nullptr) {
  using C = Cfg<R>;
  constexpr int NT = C::NT;
  const int r4 = lane >> 2, q = lane & 3;
#pragma unroll
  for (int tt = 0; tt < NT; ++tt) {
    const int ph = sPerm[8 * tt + r4];
    const double2 *kp = gK + (size_t)ph * ldkm + 8 * c + 2 * q, *mp = gM + (size_t)ph * ldkm + 8 * c + 2 * q;
    const double2 k0 = kp[0], k1 = kp[1], m0 = mp[0], m1 = mp[1];
    ar[tt][0] = fma(-s, m0.y, k0.x);
    ai[tt][0] = fma(s, m0.x, k0.y);
    ar[tt][1] = fma(-s, m1.y, k1.x);
    ai[tt][1] = fma(s, m1.x, k1.y);
  }
  constexpr bool M3 = Cfg<R, false, TM>::GAUSS3;
  double ak[NT][2];
  if constexpr (M3) {
#pragma unroll
    for (int tt = 0; tt < NT; ++tt) ak[tt][0] = ak[tt][1] = 0.0;
  }
  if constexpr (!(PODP_LL_ABLATE & 2))
    for (int b = 0; b < c; ++b)
      body_dispatch<NT, TM, M3>(b, ar, ai, ak, TM ? Sh : S, gY + (c * (c - 1) / 2 + b) * 64, lane, tm, S);
  double2 *St = TM ? S : S + strip_off<C::DIAG_L2>(NT, c) * 64;
  if constexpr (TM) __syncwarp();  // the last block's loads from the staging tile (strip tile 0) are done
#pragma unroll
  for (int tt = 0; tt < NT; ++tt) {
    if (tt >= c) {
      if constexpr (M3) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          ar[tt][e] += ak[tt][e];
          ai[tt][e] += ak[tt][e];
        }
      }
      double2 *row = St + (8 * (tt - c) + r4) * 8;
      row[(2 * q) ^ swz(r4)] = make_double2(ar[tt][0], ai[tt][0]);
      row[(2 * q + 1) ^ swz(r4)] = make_double2(ar[tt][1], ai[tt][1]);
    }
  }
}

// After the factorisation of one frequency: z = P_perm B (real-ified: cols [Re b_0..2 | Im b_0..2 | 0 0]), forward
// sweep, diagonal-block inverses D_t, block back substitution, P written (workspace and optional debug output).
template <int R, bool TM = false>
__device__ __forceinline__ void finish(const EvalArgs &a, const double *op, double om, const double2 *S,
                                       double2 *gY, double2 *gD, const double2 *gDiag, const int *sPerm, double *Pw,
                                       int64_t t, int lane, uint32_t tm = 0, const double2 *sB = nullptr,
                                       double *zt = nullptr,
                                       const double2 *Sh = nullptr) {
  using C = Cfg<R>;
  constexpr int NT = C::NT;
  const int r4 = lane >> 2, q = lane & 3;
  double z[NT][2];
  {
    // shared-memory copy: rows padded to R + 2 entries (the three directions fall into different banks)
    const int ldb = sB ? R + 2 : R;
    const double2 *gb0 = sB ? sB : reinterpret_cast<const double2 *>(op + a.L.b0);
    const double2 *gb1 = sB ? sB + 3 * (R + 2) : reinterpret_cast<const double2 *>(op + a.L.b1);
#pragma unroll
    for (int tt = 0; tt < NT; ++tt) {
      const int ph = sPerm[8 * tt + r4];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int n = 2 * q + e;
        double v = 0.0;
        if (n < 6) {
          const int d = n < 3 ? n : n - 3;
          const double2 x0 = gb0[d * ldb + ph], x1 = gb1[d * ldb + ph];
          v = n < 3 ? fma(om, x1.x, x0.x) : fma(om, x1.y, x0.y);
        }
        z[tt][e] = v;
      }
    }
  }
  if constexpr (!(PODP_LL_ABLATE & 8))
    [&]<int... Bs>(std::integer_sequence<int, Bs...>) {
      (body_rhs<NT, Bs, TM>(z, TM ? Sh : S, lane, tm, zt), ...);
    }(std::make_integer_sequence<int, NT - 1>{});
  // ---- D_t = (L_tt U_tt)^{-1}: lane -> (tile t0 + lane/8, column lane%8); stored in C-fragment order -----------
  // DIAG_L2: the strips are no longer needed after the forward sweep, so the diagonal blocks are brought back from
  // the L2 scratch into shared-memory tiles 0..NT-1 (one round of independent loads) and D_t goes to tiles
  // NT..2NT-1, where the back substitution reads it (no L2 round trips on either chain)
  // (TM: the shared-memory strip has only NT tiles; D_t overwrites the staged blocks in place, see below)
  // staged blocks and D_t sit at a stride of DS = 65 entries (the 4 blocks a pass works on then fall into different
  // 16-byte bank groups: their broadcast reads cost 1 wavefront instead of 4); the spill-over lands in sRow
  constexpr int DS = (TM && NT > 9) ? 64 : 65;
  static_assert(!TM || NT * DS <= NT * 64 + 9, "staged diagonal blocks overrun sRow");
  double2 *sD = const_cast<double2 *>(S) + (TM ? 0 : NT * DS);
  if constexpr (C::DIAG_L2 || TM) {
    __syncwarp();
    double2 *Sw = const_cast<double2 *>(S);
    for (int e = lane; e < NT * 64; e += 32) Sw[(e >> 6) * DS + (e & 63)] = __ldcg(gDiag + e);
    __syncwarp();
  }
  if constexpr (!(PODP_LL_ABLATE & 4)) {
    const int j = lane & 7;
#pragma unroll 1
    for (int t0 = 0; t0 < NT; t0 += 4) {
      const int td = t0 + (lane >> 3);
      const bool act = td < NT;
      const int tdc = act ? td : NT - 1;  // idle lanes recompute the last block (results discarded)
      {
        // L\U diagonal block of panel td: staged copy (DIAG_L2, TM) or rows 0..7 of strip td
        const double2 *Dg = (C::DIAG_L2 || TM) ? S + tdc * DS : S + strip_off<false>(NT, tdc) * 64;
        double2 y[8], x[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          double2 acc = make_double2(i == j ? 1.0 : 0.0, 0.0);
#pragma unroll
          for (int k = 0; k < i; ++k) acc = cfms(Dg[i * 8 + (k ^ swz(i))], y[k], acc);
          y[i] = acc;
        }
#pragma unroll
        for (int i = 7; i >= 0; --i) {
          double2 acc = y[i];
#pragma unroll
          for (int k = i + 1; k < 8; ++k) acc = cfms(Dg[i * 8 + (k ^ swz(i))], x[k], acc);
          x[i] = cmul(acc, Dg[i * 8 + (i ^ swz(i))]);  // 1/U_ii (stored by the panel)
        }
        double2 *dt = (C::DIAG_L2 || TM) ? sD + tdc * DS : gD + tdc * 64;
        if constexpr (TM) __syncwarp();  // D_t overwrites the staged block it was computed from
        if (act) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            if constexpr (C::DIAG_L2 || TM) dt[8 * i + (j ^ ((i & 1) << 2))] = x[i];  // see afrag_cstore_s
            else dt[2 * (4 * i + (j >> 1)) + (j & 1)] = x[i];
          }
        }
      }
    }
  }
  __syncwarp();
  // ---- block back substitution x_t = D_t (z_t - sum_{c > t} Y_tc x_c), right-looking over c -----------------
#pragma unroll
  for (int tt = NT - 1; tt >= 0; --tt) {
    double b1[2], b2[2];
    rhs_frags(z[tt][0], z[tt][1], lane, b1, b2, zt);
    const double2 d0 = (C::DIAG_L2 || TM) ? afrag_cstore_s(sD + tt * DS, 0, lane) : afrag_cstore(gD + tt * 64, 0, lane);
    const double2 d1 = (C::DIAG_L2 || TM) ? afrag_cstore_s(sD + tt * DS, 1, lane) : afrag_cstore(gD + tt * 64, 1, lane);
    double x0 = 0.0, x1 = 0.0;
    dmma(x0, x1, d0.x, b1[0]);
    dmma(x0, x1, d0.y, b2[0]);
    dmma(x0, x1, d1.x, b1[1]);
    dmma(x0, x1, d1.y, b2[1]);
    // P (3 x R complex, direction-major): column n of the real-ified tile = Re (n < 3) / Im (3 <= n < 6)
    {
      const int i = 8 * tt + r4;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int n = 2 * q + e;
        if (n < 6) {
          const int d = n < 3 ? n : n - 3, part = n < 3 ? 0 : 1;
          const double v = e ? x1 : x0;
          Pw[(d * R + i) * 2 + part] = v;
          if (a.P_out && i < a.r) a.P_out[(((size_t)t * 3 + d) * a.r + i) * 2 + part] = v;
        }
      }
    }
    if (tt > 0 && !(PODP_LL_ABLATE & 8)) {
      rhs_frags(x0, x1, lane, b1, b2, zt);
#pragma unroll
      for (int s2 = 0; s2 < 2; ++s2) {
        b1[s2] = -b1[s2];
        b2[s2] = -b2[s2];
      }
#pragma unroll
      for (int t2 = 0; t2 < tt; ++t2) {
        const double2 *gyt = gY + (tt * (tt - 1) / 2 + t2) * 64;
        const double2 y0 = afrag_cstore(gyt, 0, lane), y1 = afrag_cstore(gyt, 1, lane);
        dmma(z[t2][0], z[t2][1], y0.x, b1[0]);
        dmma(z[t2][0], z[t2][1], y0.y, b2[0]);
        dmma(z[t2][0], z[t2][1], y1.x, b1[1]);
        dmma(z[t2][0], z[t2][1], y1.y, b2[1]);
      }
    }
  }
}

// info != 0: the frequency's P is NaN (and its info code is written)
__device__ __forceinline__ void fail_out(const EvalArgs &a, double *Pw, int R, int64_t t, int info, int lane) {
  const double nanv = __longlong_as_double(0x7ff8000000000000ll);
  if (info != 0) {
    for (int e = lane; e < 6 * R; e += 32) Pw[e] = nanv;
    if (a.P_out)
      for (int e = lane; e < 6 * a.r; e += 32) a.P_out[(size_t)t * 6 * a.r + e] = nanv;
  }
  if (a.info && lane == 0) a.info[t] = info;
}

}  // namespace lull

template <int R, bool PIVOT, bool KM, bool TM = false, bool SEG = false>
__global__ void __launch_bounds__(lull::Cfg<R, KM, TM>::G * 32, 1) lu_ll_kernel(EvalArgs a) {
  using C = lull::Cfg<R, KM, TM>;
  constexpr int NT = C::NT, G = C::G;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2 *S = reinterpret_cast<double2 *>(smem_raw + (size_t)wid * C::W_BYTES);
  double2 *sRow = S + C::STRIP_TILES * 64;
  int *sPerm = reinterpret_cast<int *>(sRow + 9);
  int *sMap = sPerm + ((R + 3) / 4) * 4;  // TM: interchange source map (positions >= kb)
  // TM: 512-byte staging tile of the right-hand-side fragment conversions (rhs_frags)
  double *zt = C::ZT_BYTES ? reinterpret_cast<double *>(sMap + ((R + 3) / 4) * 4) : nullptr;
  const int64_t total = (int64_t)a.n_obj * a.F;
  const int64_t gw = (int64_t)blockIdx.x * G + wid, nw = (int64_t)gridDim.x * G;
  double2 *gY = a.gscr + (size_t)gw * C::GSCR_TILES * 64;  // Y_{t,c} at tile c(c-1)/2 + t; D_t at NT(NT-1)/2 + t
  double2 *gD = gY + (NT * (NT - 1) / 2) * 64;
  double2 *gDiag = gD + NT * 64;  // L\U diagonal blocks (panel order)
  // TM: base of the strips kept outside tensor memory (tile offsets strip_off_hyb): shared memory after the virtual
  // strip, or (HYB_G) the L2 scratch after the diagonal blocks
  double2 *Sh = C::HYB_G ? gDiag + NT * 64 - NT * 64 : S;

  double2 *sKM = reinterpret_cast<double2 *>(smem_raw + (size_t)G * C::W_BYTES);
  // TM: 512 TMEM columns for the CTA (warp 0 allocates and frees); warp w uses the lanes of its SM sub-partition
  // (32 (w % 4) ..) and columns (w / 4) TM_COLS ..
  __shared__ uint32_t s_tmem;
  uint32_t tm = 0;
  if constexpr (TM) {
    if (wid == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(&s_tmem))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    tm = s_tmem + ((uint32_t)(32 * (wid & 3)) << 16) + (uint32_t)((wid >> 2) * C::TM_COLS);
  }

  // one evaluation t = (obj, f) by this warp
  // CTA-wide rendezvous of the warps before each frequency (Cfg::LOCKSTEP); every warp of the CTA executes it the
  // same number of times (the evaluation loops below are CTA-uniform, a warp without work passes valid = false)
  auto rendezvous = [&]() {
#ifdef PODP_LL_GROUP  // dev: rendezvous within groups of PODP_LL_GROUP warps only
    asm volatile("bar.sync %0, %1;" ::"r"(1 + wid / PODP_LL_GROUP), "r"(32 * PODP_LL_GROUP) : "memory");
#else
    if constexpr (C::LOCKSTEP) __syncthreads();
#endif
  };
#ifdef PODP_LL_STAGGER  // dev: group g starts g * PODP_LL_STAGGER cycles late
  {
    const long long t0 = clock64(), wait = (long long)(wid / PODP_LL_GROUP) * PODP_LL_STAGGER;
    while (clock64() - t0 < wait) __nanosleep(200);
  }
#endif
  auto process = [&](int64_t t, int obj, int64_t f, bool valid) {
    const double *op = a.ops + (size_t)obj * a.L.stride;
    const double om = valid ? a.omega[f] : 0.0;
    const double s = om * op[a.L.scal + SC_NU];
    const double2 *gK = C::KM_BYTES ? sKM : reinterpret_cast<const double2 *>(op + a.L.K);
    const double2 *gM = C::KM_BYTES ? sKM + R * (R + 1) : reinterpret_cast<const double2 *>(op + a.L.M);
    constexpr int LDKM = C::KM_BYTES ? R + 1 : R;
    double *Pw = reinterpret_cast<double *>(a.Pws + (size_t)t * 3 * R);
    int info = valid ? (isfinite(om) ? 0 : -1) : -2;
    for (int i = lane; i < R; i += 32) sPerm[i] = i;
    __syncwarp();
    double ar[NT][2], ai[NT][2];
    for (int c = 0; c < NT; ++c) {
      if (info == 0) {
        lull::column_tile<R, TM>(c, ar, ai, S, gY, sPerm, gK, gM, s, lane, LDKM, tm, Sh);
        __syncwarp();
        if constexpr (PODP_LL_ABLATE & 1) {
          info = 0;
        } else if constexpr (C::MS > 1) {
          info = (R - 8 * c > 32) ? lull::panel<R, C::MS, PIVOT, TM>(c, S, sRow, sPerm, gDiag, lane, tm, sMap, Sh)
                                  : lull::panel<R, 1, PIVOT, TM>(c, S, sRow, sPerm, gDiag, lane, tm, sMap, Sh);
        } else {
          info = lull::panel<R, 1, PIVOT, TM>(c, S, sRow, sPerm, gDiag, lane, tm, sMap, Sh);
        }
      }
    }
    if (info == 0)
      lull::finish<R, TM>(a, op, om, S, gY, gD, gDiag, sPerm, Pw, t, lane, tm,
                          C::KM_BYTES ? sKM + 2 * R * (R + 1) : nullptr, zt, Sh);
    if (valid) lull::fail_out(a, Pw, R, t, info, lane);
    __syncwarp();
  };

  auto stage_km = [&](int obj) {  // K and M (row stride R + 1), b0 and b1 of one object -> shared memory, whole CTA
    const double *o = a.ops + (size_t)obj * a.L.stride;
    const double2 *k0p = reinterpret_cast<const double2 *>(o + a.L.K);
    const double2 *m0p = reinterpret_cast<const double2 *>(o + a.L.M);
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
      const int i = e / R, j = e - i * R;
      sKM[i * (R + 1) + j] = __ldg(k0p + e);
      sKM[R * (R + 1) + i * (R + 1) + j] = __ldg(m0p + e);
    }
    double2 *sB = sKM + 2 * R * (R + 1);
    for (int e = threadIdx.x; e < 3 * R; e += blockDim.x) {
      const int d = e / R, i = e - d * R;
      sB[d * (R + 2) + i] = __ldg(reinterpret_cast<const double2 *>(o + a.L.b0) + e);
      sB[3 * (R + 2) + d * (R + 2) + i] = __ldg(reinterpret_cast<const double2 *>(o + a.L.b1) + e);
    }
  };
  if constexpr (SEG) {
    // K and M in shared memory, several objects: the CTA takes a contiguous range of evaluations and walks it
    // object by object, staging each object's K and M once (CTA-wide barriers only at object boundaries)
    const int64_t per = (total + gridDim.x - 1) / gridDim.x;
    const int64_t start = (int64_t)blockIdx.x * per, end = start + per < total ? start + per : total;
    int64_t seg = start;
    int obj = start < total ? (int)(start / a.F) : 0;
    while (seg < end) {
      const int64_t obj_end = (int64_t)(obj + 1) * a.F, seg_end = obj_end < end ? obj_end : end;
      __syncthreads();  // every warp is done with the previous object's K and M
      stage_km(obj);
      __syncthreads();
      const int64_t fbase = (int64_t)obj * a.F;
      int it = 0;
      for (int64_t t = seg + wid; t - wid < seg_end; t += G) {
        if ((it++ & (C::LOCKSTEP_EVERY - 1)) == 0) rendezvous();
        process(t, obj, t - fbase, t < seg_end);
      }
      seg = seg_end;
      ++obj;
    }
  } else {
    // round robin over the grid's warps (one object: its K and M staged once, if KM); (obj, f) of evaluation t
    // advanced incrementally (no 64-bit division, whose subroutine call forces spills).  (Measured: for one object
    // the round robin is faster than contiguous ranges per CTA, r = 64 5.80 vs 6.17 ms.)
    if constexpr (C::KM_BYTES > 0) {
      stage_km(0);
      __syncthreads();
    }
    int obj = 0, it = 0;
    int64_t f = gw;
    while (f >= a.F) {
      f -= a.F;
      ++obj;
    }
    for (int64_t t = gw; t - wid < total; t += nw) {
      if ((it++ & (C::LOCKSTEP_EVERY - 1)) == 0) rendezvous();
      process(t, obj, f, t < total);
      f += nw;
      while (f >= a.F) {
        f -= a.F;
        ++obj;
      }
    }
  }
  if constexpr (TM) {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (wid == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(s_tmem) : "memory");
  }
}

namespace lull {
template <int R, bool KM, bool TM>
static cudaError_t launch_k(const EvalArgs &a, cudaStream_t s, int sms) {
  using C = Cfg<R, KM, TM>;
  // K and M in shared memory: contiguous per-CTA ranges walked object by object (SEG) for several objects, and for
  // one object at R <= 40 (measured: c1 solve 0.111 -> 0.104 ms); one object at 48 <= R <= 64 keeps the round robin
  // (measured faster there: r = 64 5.80 vs 6.17 ms)
  constexpr bool KMT = C::KM_BYTES > 0;
  const bool seg = KMT && (a.n_obj > 1 || KM);
  auto kern = (a.flags & PODP_FLAG_NO_PIVOT)
                  ? (seg ? lu_ll_kernel<R, false, KM, TM, KMT> : lu_ll_kernel<R, false, KM, TM, false>)
                  : (seg ? lu_ll_kernel<R, true, KM, TM, KMT> : lu_ll_kernel<R, true, KM, TM, false>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::BYTES);
  if (e != cudaSuccess) return e;
  const int64_t total = (int64_t)a.n_obj * a.F;
  int64_t blocks = (total + C::G - 1) / C::G;
  if (blocks > sms) blocks = sms;
  kern<<<(unsigned)blocks, C::G * 32, C::BYTES, s>>>(a);
  return cudaGetLastError();
}

template <int R>
static cudaError_t launch_t(const EvalArgs &a, cudaStream_t s, int sms) {
  // K and M in shared memory (per object, contiguous evaluation ranges per CTA) -- directly where it costs no warps
  // (R <= 40), with the M tiles in tensor memory for 40 < R <= 64
  if constexpr (R <= 40) {
    static_assert(Cfg<R, true>::G == Cfg<R, false>::G, "KM variant must keep the warp count");
    return launch_k<R, true, false>(a, s, sms);
  } else {
#ifndef PODP_LL_NO_TMEM
    // tensor memory where it buys warps (or, up to R = 64, K and M in shared memory)
    if constexpr (R <= 64 || Cfg<R, false, true>::G > Cfg<R, false, false>::G) return launch_k<R, false, true>(a, s, sms);
#endif
  }
  return launch_k<R, false, false>(a, s, sms);
}
}  // namespace lull

namespace lull {
template <int R>
constexpr size_t scratch_tiles() {  // per SM: the largest G x GSCR_TILES over the variants launch_t may pick
  constexpr size_t p = (size_t)Cfg<R>::G * Cfg<R>::GSCR_TILES, k = (size_t)Cfg<R, true>::G * Cfg<R, true>::GSCR_TILES;
  if constexpr (R % 8 == 0 && R >= 40) {
    constexpr size_t t = (size_t)Cfg<R, false, true>::G * Cfg<R, false, true>::GSCR_TILES;
    return (p > k ? p : k) > t ? (p > k ? p : k) : t;
  } else {
    return p > k ? p : k;
  }
}
}  // namespace lull

size_t lu_ll_scratch_bytes(int R, int sms) {
  size_t tiles = 0;
  switch (R) {
#define PODP_CASE(RR) \
  case RR: tiles = lull::scratch_tiles<RR>(); break;
    PODP_CASE(8) PODP_CASE(16) PODP_CASE(24) PODP_CASE(32) PODP_CASE(40) PODP_CASE(48) PODP_CASE(56) PODP_CASE(64)
    PODP_CASE(72) PODP_CASE(80) PODP_CASE(88) PODP_CASE(96)
#undef PODP_CASE
    default: return 0;
  }
  return (size_t)sms * tiles * 1024;
}

cudaError_t launch_lu_ll(const EvalArgs &a, cudaStream_t s, int sms) {
  if (!a.gscr) return cudaErrorInvalidValue;
  switch (a.L.R) {
#ifdef PODP_LL_ONLY_R  // dev: instantiate one size only (fast ptxas iterations)
    case PODP_LL_ONLY_R: return lull::launch_t<PODP_LL_ONLY_R>(a, s, sms);
#else
    case 8: return lull::launch_t<8>(a, s, sms);
    case 16: return lull::launch_t<16>(a, s, sms);
    case 24: return lull::launch_t<24>(a, s, sms);
    case 32: return lull::launch_t<32>(a, s, sms);
    case 40: return lull::launch_t<40>(a, s, sms);
    case 48: return lull::launch_t<48>(a, s, sms);
    case 56: return lull::launch_t<56>(a, s, sms);
    case 64: return lull::launch_t<64>(a, s, sms);
    case 72: return lull::launch_t<72>(a, s, sms);
    case 80: return lull::launch_t<80>(a, s, sms);
    case 88: return lull::launch_t<88>(a, s, sms);
    case 96: return lull::launch_t<96>(a, s, sms);
#endif
    default: return cudaErrorNotSupported;
  }
}

}  // namespace podp
