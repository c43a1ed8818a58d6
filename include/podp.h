/* podp.h -- C ABI of libpodp: the on-line stage of projected POD (PODP) for magnetic polarizability tensor
 * (MPT) spectral signatures, arXiv 2307.05590 (Elgy & Ledger), on one NVIDIA B200 (sm_100a), FP64.
 *
 * Citations: "P:<line>" = PAPER.md (the paper's LaTeX), with the section / equation label it falls in.
 *
 * What one evaluation computes, for every output frequency omega (Algorithm 1 lines 22-26):
 *   a2  A(omega) = K + i*omega*nu*M,  B(omega) = b0 + omega*b1            (eqn:ReducedA; BASELINE sign)
 *   a3  P(omega) = A(omega)^{-1} B(omega)  (r x 3; column i = p_i)        (eqn:ReducedA)
 *   a4  R_ij = -(alpha^3/4) Re(p_i^H K_R p_j),  Rt = N0 + R               (eqn:podprealmpt P:600-604; eqn:NRI P:440)
 *       I_ij = (omega alpha^3/4) (S_ij + nu Re(p_i^H M p_j) + Re(h_i p_j) + Re(h_j p_i))
 *                                                                          (eqn:podpimagmpt P:606-620, shared basis)
 *   a5  X_ij = w_i^H G w_j with w_i = [e_{2i} + omega e_{2i+1} | -p_i | -i omega nu p_i]
 *       n_i = max(0, Re X_ii), m_ij = max(0, n_i + n_j - 2 Re X_ij),
 *       Delta_ij = alpha^3/(8 alpha_LB) (n_i + n_j + m_ij)                 (lemma:certificate)
 *   a6  outputs: Rt (or R), I, Delta as F x 6 row-major doubles, entry order (11,22,33,12,13,23)
 *   a7  podp_select: one greedy step of Algorithm 1
 *
 * Conventions (all functions):
 *   - complex = interleaved (re, im) double pairs, i.e. C99 double _Complex / numpy complex128 /
 *     torch.complex128.  Declared here as `const double *` pointing at 2*n doubles.
 *   - ALL matrices are ROW-MAJOR (C order), matching NumPy/PyTorch.  A Hermitian matrix passed transposed
 *     arrives as its conjugate and silently conjugates the results (SURVEY "layout trap"); there is no check.
 *   - No function aborts, throws or exits across the ABI.  Every non-OK status sets a thread-local message
 *     readable with podp_last_error().
 *   - "device" pointers are CUDA device pointers on the context's device; "host" pointers are CPU memory
 *     (pinned memory makes the host-buffer entry points faster but is not required).
 *   - cuda_stream is a cudaStream_t (NULL = legacy default stream).
 */
#ifndef PODP_H
#define PODP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PODP_R_MAX 128          /* largest supported number of POD modes r (configs need <= 96) */
#define PODP_SNAP_MAX 1025      /* largest snapshot set accepted by podp_select (<= 1024 intervals) */

typedef struct podp_ctx podp_ctx; /* opaque; owns packed device copies of the operators; read-only after create */

typedef enum {
  PODP_OK = 0,
  PODP_ERR_ARG = 1,           /* invalid argument (null pointer, r out of range, F < 0, nu/alpha/alpha_lb <= 0, ...) */
  PODP_ERR_CUDA = 2,          /* a CUDA runtime call or kernel launch failed */
  PODP_ERR_OOM = 3,           /* device or pinned-host allocation failed */
  PODP_ERR_UNSUPPORTED = 4,   /* e.g. device is not sm_100 */
  PODP_ERR_NONFINITE = 5,     /* a non-finite value in an operator input */
  PODP_ERR_NOT_HERMITIAN = 6, /* K, M, K_R or G has a Hermitian defect above 1e-12 * max|X| */
  PODP_ERR_NO_CANDIDATES = 7  /* podp_select: fewer non-empty intervals than requested */
} podp_status;

enum {
  PODP_FLAG_DEFAULT = 0,        /* first output = Rt = N0 + R                                              */
  PODP_FLAG_OUT_R = 1u << 0,    /* first output = omega-dependent R only (used by parity runs, reading U11)  */
  PODP_FLAG_OUT_P = 1u << 1,    /* debug: also write P (n_obj x F x 3 x r complex, row-major) to P_d       */
  PODP_FLAG_NO_PIVOT = 1u << 2, /* LU without pivoting (exists since Re x^H A x = x^H K x > 0 for K > 0;
                                   SURVEY Appendix A.4).  Default is partial pivoting.                       */
  PODP_FLAG_PENCIL = 1u << 3,   /* NEXT row N3: solve with the pencil reduction precomputed by
                                   podp_create (K = L L^H, L^{-1} M L^{-H} = V Lambda V^H, Z = L^{-H} V), i.e.
                                   P = Z (I + i omega nu Lambda)^{-1} Z^H B(omega): O(r^2) per frequency instead of
                                   the LU's O(r^3).  Exact in exact arithmetic; requires K positive definite
                                   (PODP_ERR_UNSUPPORTED otherwise).  R, I, Delta are then formed as usual.
                                   The precompute runs once, on the first evaluation that asks for it.        */
  /* Solver selection, for A/B measurement (at most one; none = the measured default: PODP_FLAG_LU_LL for padded
     r <= 96, PODP_FLAG_LU_GENERIC above).  Every choice computes the same
     pivoted LU solve of P:593-596 up to rounding; a choice not instantiated for this r -> PODP_ERR_UNSUPPORTED. */
  PODP_FLAG_LU_LL = 1u << 8,      /* left-looking block LU, one warp per frequency, padded r <= 96 (k_lu_ll.cu) */
  PODP_FLAG_LU_BLK = 1u << 9,     /* lock-step panel-blocked LU, W warps per frequency, padded r <= 96        */
  PODP_FLAG_LU_DYN = 1u << 10,    /* dynamically scheduled blocked LU, W warps per frequency, padded r <= 96  */
  PODP_FLAG_LU_GENERIC = 1u << 11, /* generic one-warp LU (any r <= 128, pivoting or PODP_FLAG_NO_PIVOT)      */
  /* Measurement only (A/B of the contraction design): the MPT / certificate forms as FP64 tensor-core GEMMs over the
     solution panel with bulk-copy (TMA) staging (k_mpt_gemm.cu) instead of the default operator-stationary kernel;
     one object, padded r in {24, 48, 96}, not with PODP_FLAG_PENCIL (else PODP_ERR_UNSUPPORTED).  Same results up
     to rounding. */
  PODP_FLAG_MPT_GEMM = 1u << 13,
  /* Measurement only (A/B): the contraction kernel with two frequencies per lane (halves the shared-memory operator
     traffic, + 13 % executed flops; measured slower: 1.00 vs 0.94 ms per 1e5 at r = 48); one object, padded r = 48,
     not with PODP_FLAG_PENCIL, PODP_FLAG_MPT_GEMM or the per-direction form (else PODP_ERR_UNSUPPORTED; the
     per-direction form ignores it).  Same results up to rounding. */
  PODP_FLAG_MPT_PAIR = 1u << 14
};

/* Operators of ONE object (host pointers; copied, validated and packed by podp_create; caller keeps ownership).
 * r = number of POD modes (paper's M).  Shared reduced basis (BASELINE reading U3). */
typedef struct {
  int32_t r;            /* 1 <= r <= PODP_R_MAX                                                                 */
  double nu;            /* mu0*sigma*alpha^2 > 0, omega-free (paper's nu-tilde)                           */
  double alpha;         /* object size alpha > 0; enters as alpha^3/4 and alpha^3/(8 alpha_LB)                   */
  double alpha_lb;      /* stability lower bound alpha_LB > 0 (lemma:certificate)                        */
  const double *K;      /* r x r complex Hermitian: reduced system stiffness (incl. eps*M_reg)            */
  const double *M;      /* r x r complex Hermitian PSD: nu-free reduced conductor mass (C^M / nu)         */
  const double *K_R;    /* r x r complex Hermitian, or NULL (= K): stiffness used in R (reading U4)             */
  const double *b0;     /* r x 3 complex (row-major; column i = direction i): omega^0 part of r_i^M (reading U2) */
  const double *b1;     /* r x 3 complex: omega^1 part of r_i^M                                                  */
  const double *N0;     /* 3 x 3 real symmetric: N^0 (omega-independent)                           */
  const double *S;      /* 3 x 3 real symmetric: o_i^T C1 o_j + c_ij + s_i^T o_j + s_j^T o_i  */
  const double *H;      /* 3 x r complex: row i = h_i = o_i^T C2 U + t_i^T U (unconjugated)           */
  const double *G;      /* (6+2r) x (6+2r) complex Hermitian PSD Gram of the residual factor, slot order
                           [b0_1, b1_1, b0_2, b1_2, b0_3, b1_3 | K U (r) | M U (r)]  (reading U9)     */
  const double *M_I;    /* r x r complex Hermitian, or NULL (= M): conductor mass used in I only.  The paper's
                           per-direction form (NEXT row N1; U_i^M per direction) is the
                           embedding U = [U_1 U_2 U_3] (r = M_1+M_2+M_3) with K, M block-diagonal (A_i^M blocks,
                           P:596), b0/b1 column i nonzero only in block i, K_R = [K_ij^M], M_I = [C_ij^M]/nu
                           (P:618), H row i = [o_i^T C2 U_j + t_i U_j]_j and G the Gram of
                           [B0_1, B1_1, ..., B1_3 | K U | M U]; then column i of P is (0, p_i^M, 0).         */
} podp_operators;

/* Validate + pack one object's operators onto `device`; the upload is enqueued on cuda_stream and complete
 * when podp_create returns.  Returns PODP_ERR_ARG / _NONFINITE / _NOT_HERMITIAN / _OOM / _CUDA / _UNSUPPORTED. */
podp_status podp_create(const podp_operators *ops, int device, void *cuda_stream, podp_ctx **out);

/* Same for n_obj >= 1 independent objects (dictionary batch, BASELINE config 3); all must share r. */
podp_status podp_create_batch(int32_t n_obj, const podp_operators *ops, int device, void *cuda_stream,
                              podp_ctx **out);

/* NEXT row N1 in the paper's LITERAL per-direction form (P:584 U_i^M per direction with M_i modes; P:593-596
 * eqn:ReducedA, one reduced system A_i^M p_i = r_i^M of size M_i per direction; P:600-604 eqn:podprealmpt and
 * P:606-620 eqn:podpimagmpt with the rectangular cross blocks K_ij^M, C_ij^M, h_i^(j); P:651-661 the certificate
 * from the direction Grams G_ij = W_i^H W_j, W_i = [B0_i, B1_i | K U_i | M U_i]).  All pointers host, complex =
 * interleaved (re, im) doubles, row-major; copied by podp_create_perdir; caller keeps ownership. */
typedef struct {
  int32_t m[3];         /* M_1, M_2, M_3 >= 1 with M_1 + M_2 + M_3 <= PODP_R_MAX                                 */
  double nu, alpha, alpha_lb;                   /* as in podp_operators                                          */
  const double *K[9];   /* K[3i+j]: M_i x M_j complex, K_ij^M = U_i^H K U_j; K[3i+i] Hermitian (the direction-i
                           system stiffness); all nine blocks enter R_ij                          */
  const double *C[9];   /* C[3i+j]: M_i x M_j complex, C_ij^M / nu = U_i^H M U_j; C[3i+i] Hermitian PSD (the
                           direction-i conductor mass); all nine enter I_ij                       */
  const double *b0[3];  /* b0[i]: M_i complex, omega^0 part of r_i^M (reading U2)                                */
  const double *b1[3];  /* b1[i]: M_i complex, omega^1 part                                                       */
  const double *H[9];   /* H[3i+j]: M_j complex, row h_i^(j) = o_i^T C2 U_j + t_i U_j (unconjugated)       */
  const double *N0;     /* 3 x 3 real symmetric                                                                  */
  const double *S;      /* 3 x 3 real symmetric                                                      */
  const double *G[9];   /* G[3i+j]: (2+2M_i) x (2+2M_j) complex, W_i^H W_j with W_i's slot order
                           [B0_i, B1_i | K U_i (M_i) | M U_i (M_i)]; G[3i+j] = G[3j+i]^H                        */
} podp_perdir_operators;

/* Validate + pack the literal per-direction operators.  podp_eval on the returned context solves the THREE
 * direction systems (sizes M_1, M_2, M_3: three batched LU solves per omega instead of one of size sum M_i) and
 * evaluates R, I and Delta from the cross blocks; outputs, info (k+1 for a zero pivot at step k of the
 * concatenated columns, i.e. M_1 + ... + M_{i-1} + k_i + 1 for direction i) and podp_select are as for podp_eval,
 * and PODP_FLAG_OUT_P returns P as 3 x (M_1+M_2+M_3) with column i = (0, p_i^M, 0).  PODP_FLAG_PENCIL is
 * PODP_ERR_UNSUPPORTED on such a context.  Errors as podp_create. */
podp_status podp_create_perdir(const podp_perdir_operators *ops, int device, void *cuda_stream, podp_ctx **out);

/* Device-buffer evaluation (the hot path).  Asynchronous on cuda_stream; no host synchronisation.
 *   omega_d : device, F doubles (the same output grid for every object)
 *   T1_d    : device, n_obj x F x 6 doubles: Rt = N0 + R (default) or R (PODP_FLAG_OUT_R)
 *   I_d     : device, n_obj x F x 6 doubles
 *   Delta_d : device, n_obj x F x 6 doubles
 *   info_d  : device, n_obj x F int32, nullable: 0 = ok; k+1 = exactly-zero pivot at step k (LAPACK getrf
 *             convention); -1 = non-finite omega.  Failed rows of T1/I/Delta are NaN; other rows unaffected.
 *   P_d     : device, n_obj x F x 3 x r complex (only read if PODP_FLAG_OUT_P, else may be NULL)
 * F == 0 is a no-op.  Outputs are caller-owned; the context is not modified (concurrent evals on different
 * streams with distinct outputs are safe). */
podp_status podp_eval(const podp_ctx *ctx, const double *omega_d, int64_t F, double *T1_d, double *I_d,
                      double *Delta_d, int32_t *info_d, double *P_d, int flags, void *cuda_stream);

/* Host-buffer evaluation (the end-to-end entry point): copies omega host->device, runs podp_eval, copies the
 * outputs device->host and synchronises cuda_stream before returning.  Same shapes as podp_eval, all host.
 * For one object and F >= 8192 the contraction runs as two launches over the halves of the frequency range and the
 * first half's rows are copied back on a copy stream owned by the context while the second half is computed (same
 * results bit for bit).  Host evaluations of one context are serialised among themselves (they share that stream);
 * pinned host buffers make the copies asynchronous, pageable ones work too. */
podp_status podp_eval_host(const podp_ctx *ctx, const double *omega_h, int64_t F, double *T1_h, double *I_h,
                           double *Delta_h, int32_t *info_h, int flags, void *cuda_stream);

/* One greedy step of Algorithm 1 (P:677-682 lines 10-15) on object `obj` of the context's layout:
 *   intervals [snap_n, snap_{n+1}), n = 0..n_snap-2, the last one closed (reading U12); grid points equal to a
 *   snapshot or outside [snap_0, snap_{n_snap-1}] are not candidates; NaN Delta entries are ignored.
 *   Lambda_n = max over in-interval omega and the 6 entries of Delta; argmax = lowest grid index among ties.
 *   theta <= 0: choose the n_star intervals with the largest Lambda_n (ties -> lower n);
 *   0 < theta <= 1: choose intervals with Lambda_n >= theta * Lambda (at most n_star, largest first).
 *   omega_d, Delta_d: device (F and F x 6 doubles, e.g. podp_eval outputs for that object);
 *   snap_omega: host, strictly ascending, 2 <= n_snap <= PODP_SNAP_MAX;
 *   outputs (host): *n_new chosen (<= n_star), omega_new[n_star] ascending, idx_new[n_star] grid indices,
 *   *Lambda global max, Lambda_n[n_snap-1] per-interval maxima (nullable; -1 for empty intervals).
 *   Synchronises cuda_stream.  PODP_ERR_NO_CANDIDATES if theta <= 0 and fewer than n_star intervals are non-empty
 *   (or no interval is non-empty). */
podp_status podp_select(const podp_ctx *ctx, const double *omega_d, const double *Delta_d, int64_t F,
                        const double *snap_omega, int32_t n_snap, int32_t n_star, double theta, int32_t *n_new,
                        double *omega_new, int64_t *idx_new, double *Lambda, double *Lambda_n,
                        void *cuda_stream);

/* NEXT row N4 -- per-frequency epilogues on podp_eval outputs (device buffers, asynchronous):
 *   podp_invariants: eigenvalues of Rt (first output) and of I, ascending, n x 3 doubles each -- the rotation
 *     invariants used for dictionary matching.  n = number of output rows (n_obj * F).
 *   podp_coil_voltage: V_c = (H0^ms_c)_i (Rt + i I)_ij (H0_c)_j for n_coil coil pairs (eqn:meas_voltage,
 *     P:393-395).  h_ex, h_ms: host, n_coil x 3 real background fields at the object; V_d: device, n x n_coil
 *     complex (interleaved re, im).  1 <= n_coil <= 64.  Synchronous w.r.t. the small host->device copy only. */
podp_status podp_invariants(const double *T1_d, const double *I_d, int64_t n, double *eigR_d, double *eigI_d,
                            void *cuda_stream);
podp_status podp_coil_voltage(const double *T1_d, const double *I_d, int64_t n, const double *h_ex,
                              const double *h_ms, int32_t n_coil, double *V_d, void *cuda_stream);

/* Number of objects / modes of a context (0 if ctx is NULL). */
int32_t podp_n_obj(const podp_ctx *ctx);
int32_t podp_r(const podp_ctx *ctx);

/* Number of kernel launches the last podp_eval on this thread enqueued (bench bookkeeping). */
int32_t podp_last_launch_count(void);

/* Benchmark instrumentation.  While enabled (on != 0), podp_eval / podp_select record a CUDA event pair on the
 * caller's stream around each kernel they launch ("solve", "mpt", "select").  podp_profile_read accumulates the
 * elapsed time of every recorded pair per kernel name; call it only after the streams used are idle (it calls
 * cudaEventSynchronize on each pair).  names: n x 32 chars (NUL-terminated), ms/counts: n entries.
 * Returns the number of distinct names written (<= max_entries); reset != 0 clears the accumulators. */
podp_status podp_profile_enable(int on);
int32_t podp_profile_read(char *names, double *ms, int64_t *counts, int32_t max_entries, int32_t reset);

/* Release a context (NULL-safe; synchronises the device work that used it is the caller's job). */
podp_status podp_destroy(podp_ctx *ctx);

/* Thread-local message of the last non-OK status ("" if none). */
/* Workspace memory (the P hand-off, LU and select scratch) comes from one stream-ordered pool per device that the
 * library keeps for the process lifetime, so evaluations reuse mapped memory across calls and contexts.  This
 * returns the pool's unused memory to the driver (cudaMemPoolTrimTo 0); safe at any time (in-flight evaluations keep
 * their allocations).  PODP_OK, or PODP_ERR_ARG for a device the library has not used. */
podp_status podp_release_workspace(int device);

const char *podp_last_error(void);

/* Library version string. */
const char *podp_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PODP_H */
