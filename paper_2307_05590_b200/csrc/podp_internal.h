// Internal declarations shared by the libpodp translation units (not part of the C ABI).
#pragma once
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#include "podp.h"

namespace podp {

// Packed per-object operator layout on the device (all doubles; complex = (re, im) pairs; row-major).
// Built by podp_create (podp_api.cu) from the C-ABI inputs.  R = padded mode count (exact padding:
// K_pad = diag(K, I), everything else zero-padded; SURVEY 7 "Padding r ... is exact").
struct Layout {
  int R;          // padded r
  int64_t K, M, KR, MI, Gkk, J, Gmm;  // R x R complex (MI: mass in I; = M unless per-direction, N1)
  int64_t b0, b1, H;              // 3 x R complex (direction-major: b0[c*R + i] = b0_user[i][c])
  int64_t GbK, GbM;               // 6 x R complex (row a = b-slot a)
  int64_t Gbb;                    // 6 x 6 complex
  int64_t scal;                   // SCAL_N doubles (see below)
  int64_t Z, lam, c0, c1;         // pencil precompute (N3): Z (R x R complex), lambda (R), c0, c1 (3 x R complex)
  // N3 operators in the pencil coordinates y (P = Z y): X~ = Z^H X Z for K_R, M_I, G_KK, J, G_MM; H~ = H Z;
  // G~_bK = G_bK Z, G~_bM = G_bM Z.  The MPT/certificate kernel runs on y with these unchanged.
  int64_t PKR, PMI, PGkk, PJ, PGmm, PH, PGbK, PGbM;
  int64_t stride;                 // doubles per object (multiple of 32)
};

enum { SC_NU = 0, SC_ALPHA = 1, SC_ALPHA_LB = 2, SC_PENCIL_OK = 3, SC_S = 4, SC_N0 = 13, SC_PENCIL_DIAG = 22, SCAL_N = 32 };

Layout make_layout(int R);

struct EvalArgs {
  const double *ops;   // packed operators, n_obj objects
  Layout L;
  int r;               // true r (for the P debug output)
  int n_obj;
  const double *omega; // F
  int64_t F;
  double *T1, *I, *Delta;
  int32_t *info;
  double *P_out;       // debug P (nullable)
  double2 *Pws;        // workspace: n_obj x F x 3 x R complex (solve -> contraction hand-off)
  double2 *gscr;       // LU scratch (kernel-specific size, see the *_scratch_bytes functions), nullable
  int flags;
  int blk_hi[2];       // N1 literal form: ends of direction blocks 0 and 1 in the concatenated rows (SL-aligned);
                       // blk_hi[0] == 0 for the shared-basis form
};

// Kernel launchers (return cudaGetLastError() after the launch; cudaErrorNotSupported if no instantiation).
cudaError_t launch_lu_ll(const EvalArgs &a, cudaStream_t s, int sms);  // R <= 64, one warp per frequency
size_t lu_ll_scratch_bytes(int R, int sms);                           // its per-warp L2 scratch (Y_tc, D_t)
cudaError_t launch_lu_blk(const EvalArgs &a, cudaStream_t s);
cudaError_t launch_lu_dyn(const EvalArgs &a, cudaStream_t s);
size_t lu_dyn_scratch_bytes(int R, int sms);                          // right-hand-side scratch of its RG mode
cudaError_t launch_mpt_tile(const EvalArgs &a, cudaStream_t s, bool diag = false);
cudaError_t launch_mpt_gemm(const EvalArgs &a, cudaStream_t s, int sms);  // A/B: DMMA GEMM + bulk-copy variant
cudaError_t launch_pencil(const EvalArgs &a, cudaStream_t s);    // N3 pencil solve (P only)
cudaError_t launch_pencil_y(const EvalArgs &a, cudaStream_t s);  // N3: y = (I + i s Lambda)^{-1}(c0 + omega c1) only
cudaError_t launch_invariants(const double *T1, const double *I, int64_t n, double *eigR, double *eigI, cudaStream_t s);
cudaError_t launch_coil_voltage(const double *T1, const double *I, int64_t n, const double *hex_d, const double *hms_d,
                                int n_coil, double *V, cudaStream_t s);
bool pencil_precompute(int r, const double *K, const double *M, const double *b0, const double *b1,
                       std::vector<double> &Z, std::vector<double> &lam, std::vector<double> &c0,
                       std::vector<double> &c1);
cudaError_t launch_solve(const EvalArgs &a, cudaStream_t s, double2 *gscratch);  // generic: any R, pivot or not
size_t solve_scratch_bytes(int R, int sms);  // global scratch launch_solve needs for this R (0 if shared fits)
cudaError_t launch_perdir_scatter(const double2 *const Pd[3], const int Rs[3], const int m[3], const int offp[3],
                                  const int32_t *info3, int64_t F, double2 *Pe, int Re, int32_t *info, double *P_out,
                                  cudaStream_t s);
cudaError_t launch_select(const double *omega, const double *Delta, int64_t F, const double *snap_d, int n_snap,
                          int n_star, double theta, unsigned long long *lam_bits, unsigned long long *arg_idx,
                          double *result_d, cudaStream_t s, int *nlaunch);

}  // namespace podp
