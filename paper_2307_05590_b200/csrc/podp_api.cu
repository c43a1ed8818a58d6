// libpodp C ABI (include/podp.h): validation, packing (row a1 of SURVEY 8(a)), launch orchestration.
// Host-side only; kernels live in k_lu_ll.cu (default a2-a3; A/B: k_lu_blk.cu, k_lu_dyn.cu, generic k_solve.cu),
// k_mpt_tile.cu (a4-a6), k_select.cu (a7), k_pencil.cu (N3), k_perdir.cu (N1), k_epilogue.cu (N4).
#include <cmath>
#include <complex>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>
#include <mutex>

#include "podp_internal.h"

struct podp_ctx {
  int device;
  int r;
  int n_obj;
  int sms;
  podp::Layout L;
  double *d_ops;
  cudaMemPool_t pool;  // stream-ordered scratch (P hand-off workspace, LU scratch); keeps memory mapped between calls
  // N3 pencil precompute, done lazily by the first PODP_FLAG_PENCIL evaluation (podp_create stays O(r^2) per object)
  std::vector<double> hK, hM, hb0, hb1;  // per object: r x r, r x r, r x 3, r x 3 complex (host copies)
  std::vector<char> has_KR_MI;           // per object: K_R or M_I given (pencil coordinates not diagonal)
  std::mutex pencil_mu;
  bool pencil_done = false;
  bool pencil_ok = false;    // K positive definite for every object
  bool pencil_diag = false;  // every object has K_R = K and M_I = M: Z^H K_R Z = I, Z^H M_I Z = Lambda exactly
  // N1 literal per-direction form (podp_create_perdir): this context holds the concatenated cross-block operators
  // used by the contraction kernel; dir[i] holds direction i's system (M_i modes, padded to 8 ceil(M_i / 8)),
  // factored by its own solve launch
  // podp_eval_host: copy stream and events of the overlapped device-to-host copy (created on first use)
  std::mutex host_mu;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_half = nullptr, ev_copied = nullptr;
  podp_ctx *dir[3] = {nullptr, nullptr, nullptr};
  int m[3] = {0, 0, 0};
  int offp[3] = {0, 0, 0};  // direction block offsets in the padded (SL-aligned) concatenation
};

namespace {

thread_local std::string g_err;

// podp_eval_host -> podp_eval: host destinations of the outputs.  When set (one object, default contraction kernel,
// F >= 2 * HOST_SPLIT_MIN), the contraction runs as two launches over the halves of the frequency range and the first
// half's rows are copied to the host on the context's copy stream while the second half is computed; F1 returns the
// number of frequencies already copied.
struct HostSplit {
  double *T1_h, *I_h, *D_h;
  cudaStream_t cs;
  cudaEvent_t ev;
  int64_t F1;
};
thread_local HostSplit *g_split = nullptr;
constexpr int64_t HOST_SPLIT_MIN = 4096;

// ---- benchmark instrumentation (podp_profile_*) ---------------------------------------------------------------
struct ProfPair {
  const char *name;
  cudaEvent_t a, b;
};
bool g_prof_on = false;
std::vector<ProfPair> g_prof_pending;
std::vector<std::pair<std::string, std::pair<double, int64_t>>> g_prof_acc;

struct ProfScope {
  cudaEvent_t a = nullptr, b = nullptr;
  const char *name;
  cudaStream_t s;
  ProfScope(const char *n, cudaStream_t st) : name(n), s(st) {
    if (!g_prof_on) return;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s);
  }
  ~ProfScope() {
    if (!a) return;
    cudaEventRecord(b, s);
    g_prof_pending.push_back({name, a, b});
  }
};
thread_local int g_last_launches = 0;

podp_status fail(podp_status st, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

podp_status cuda_fail(cudaError_t e, const char *what) {
  cudaGetLastError();  // clear sticky-free errors
  if (e == cudaErrorMemoryAllocation) return fail(PODP_ERR_OOM, "%s: %s", what, cudaGetErrorString(e));
  return fail(PODP_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

// Saves/restores the caller's current device.
struct DeviceGuard {
  int prev = -1;
  bool ok = false;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    ok = cudaSetDevice(dev) == cudaSuccess;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

bool all_finite(const double *x, size_t n) {
  for (size_t i = 0; i < n; ++i)
    if (!std::isfinite(x[i])) return false;
  return true;
}

// Hermitian defect max|X - X^H| <= 1e-12 max|X| (SURVEY 8(b) "Errors")
bool is_hermitian(const double *X, int n) {
  double mx = 0.0, defect = 0.0;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      const double re = X[2 * (i * n + j)], im = X[2 * (i * n + j) + 1];
      mx = std::fmax(mx, std::hypot(re, im));
      const double tre = X[2 * (j * n + i)], tim = -X[2 * (j * n + i) + 1];
      defect = std::fmax(defect, std::hypot(re - tre, im - tim));
    }
  return defect <= 1e-12 * mx;
}

bool is_symmetric3(const double *X) {
  double mx = 0.0, defect = 0.0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      mx = std::fmax(mx, std::fabs(X[i * 3 + j]));
      defect = std::fmax(defect, std::fabs(X[i * 3 + j] - X[j * 3 + i]));
    }
  return defect <= 1e-12 * mx;
}

podp_status validate(const podp_operators &o, int idx) {
  if (o.r < 1 || o.r > PODP_R_MAX) return fail(PODP_ERR_ARG, "object %d: r=%d out of range [1,%d]", idx, o.r, PODP_R_MAX);
  if (!o.K || !o.M || !o.b0 || !o.b1 || !o.N0 || !o.S || !o.H || !o.G)
    return fail(PODP_ERR_ARG, "object %d: null operator pointer", idx);
  if (!(o.nu > 0.0) || !std::isfinite(o.nu)) return fail(PODP_ERR_ARG, "object %d: nu must be finite and > 0", idx);
  if (!(o.alpha > 0.0) || !std::isfinite(o.alpha)) return fail(PODP_ERR_ARG, "object %d: alpha must be finite and > 0", idx);
  if (!(o.alpha_lb > 0.0) || !std::isfinite(o.alpha_lb))
    return fail(PODP_ERR_ARG, "object %d: alpha_lb must be finite and > 0", idx);
  const int r = o.r, ng = 6 + 2 * r;
  const size_t rr = (size_t)2 * r * r;
  if (!all_finite(o.K, rr) || !all_finite(o.M, rr) || (o.K_R && !all_finite(o.K_R, rr)) || (o.M_I && !all_finite(o.M_I, rr)) ||
      !all_finite(o.b0, 6 * (size_t)r) || !all_finite(o.b1, 6 * (size_t)r) || !all_finite(o.N0, 9) ||
      !all_finite(o.S, 9) || !all_finite(o.H, 6 * (size_t)r) || !all_finite(o.G, (size_t)2 * ng * ng))
    return fail(PODP_ERR_NONFINITE, "object %d: non-finite operator entry", idx);
  if (!is_hermitian(o.K, r)) return fail(PODP_ERR_NOT_HERMITIAN, "object %d: K is not Hermitian", idx);
  if (!is_hermitian(o.M, r)) return fail(PODP_ERR_NOT_HERMITIAN, "object %d: M is not Hermitian", idx);
  if (o.K_R && !is_hermitian(o.K_R, r)) return fail(PODP_ERR_NOT_HERMITIAN, "object %d: K_R is not Hermitian", idx);
  if (o.M_I && !is_hermitian(o.M_I, r)) return fail(PODP_ERR_NOT_HERMITIAN, "object %d: M_I is not Hermitian", idx);
  if (!is_hermitian(o.G, ng)) return fail(PODP_ERR_NOT_HERMITIAN, "object %d: G is not Hermitian", idx);
  if (!is_symmetric3(o.S) || !is_symmetric3(o.N0)) return fail(PODP_ERR_ARG, "object %d: S / N0 not symmetric", idx);
  return PODP_OK;
}

// N3: operators in pencil coordinates (P = Z y).  Quadratic forms p_i^H X p_j = y_i^H (Z^H X Z) y_j and linear
// forms h p = (h Z) y, so the MPT/certificate kernel runs unchanged on y with X~ = Z^H X Z, H~ = H Z,
// G~_bK = G_bK Z, G~_bM = G_bM Z (all already padded to R; Z_pad = diag(Z, I)).
void pencil_transform(const podp::Layout &L, double *dst) {
  using cd = std::complex<double>;
  const int R = L.R;
  auto at = [&](int64_t base, int ld, int i, int j) { return cd(dst[base + 2 * ((size_t)i * ld + j)], dst[base + 2 * ((size_t)i * ld + j) + 1]); };
  std::vector<cd> Z((size_t)R * R), T((size_t)R * R);
  for (int i = 0; i < R; ++i)
    for (int j = 0; j < R; ++j) Z[(size_t)i * R + j] = at(L.Z, R, i, j);
  const int64_t src[5] = {L.KR, L.MI, L.Gkk, L.J, L.Gmm}, dstb[5] = {L.PKR, L.PMI, L.PGkk, L.PJ, L.PGmm};
  for (int q = 0; q < 5; ++q) {
    for (int i = 0; i < R; ++i)  // T = X Z
      for (int j = 0; j < R; ++j) {
        cd acc = 0.0;
        for (int k = 0; k < R; ++k) acc += at(src[q], R, i, k) * Z[(size_t)k * R + j];
        T[(size_t)i * R + j] = acc;
      }
    for (int i = 0; i < R; ++i)  // Z^H T
      for (int j = 0; j < R; ++j) {
        cd acc = 0.0;
        for (int k = 0; k < R; ++k) acc += std::conj(Z[(size_t)k * R + i]) * T[(size_t)k * R + j];
        dst[dstb[q] + 2 * ((size_t)i * R + j)] = acc.real();
        dst[dstb[q] + 2 * ((size_t)i * R + j) + 1] = acc.imag();
      }
  }
  const int64_t vs[3] = {L.H, L.GbK, L.GbM}, vd[3] = {L.PH, L.PGbK, L.PGbM};
  const int rows[3] = {3, 6, 6};
  for (int q = 0; q < 3; ++q)
    for (int a = 0; a < rows[q]; ++a)
      for (int j = 0; j < R; ++j) {
        cd acc = 0.0;
        for (int k = 0; k < R; ++k) acc += at(vs[q], R, a, k) * Z[(size_t)k * R + j];
        dst[vd[q] + 2 * ((size_t)a * R + j)] = acc.real();
        dst[vd[q] + 2 * ((size_t)a * R + j) + 1] = acc.imag();
      }
}

// Pack one object into dst (L.stride doubles, zero-initialised by the caller).
void pack(const podp_operators &o, const podp::Layout &L, double *dst) {
  const int r = o.r, R = L.R, ng = 6 + 2 * r;
  auto C = [](const double *X, int ld, int i, int j, int comp) { return X[2 * ((size_t)i * ld + j) + comp]; };
  for (int i = 0; i < R; ++i)
    for (int j = 0; j < R; ++j) {
      const bool in = i < r && j < r;
      for (int c = 0; c < 2; ++c) {
        const size_t e = 2 * ((size_t)i * R + j) + c;
        dst[L.K + e] = in ? C(o.K, r, i, j, c) : (i == j && c == 0 ? 1.0 : 0.0);  // K_pad = diag(K, I)
        dst[L.M + e] = in ? C(o.M, r, i, j, c) : 0.0;
        dst[L.KR + e] = in ? C(o.K_R ? o.K_R : o.K, r, i, j, c) : 0.0;
        dst[L.MI + e] = in ? C(o.M_I ? o.M_I : o.M, r, i, j, c) : 0.0;
        dst[L.Gkk + e] = in ? C(o.G, ng, 6 + i, 6 + j, c) : 0.0;
        dst[L.Gmm + e] = in ? C(o.G, ng, 6 + r + i, 6 + r + j, c) : 0.0;
      }
      // J = i (G_KM - G_MK): re = -(Im G_KM - Im G_MK), im = Re G_KM - Re G_MK
      if (in) {
        const double kmr = C(o.G, ng, 6 + i, 6 + r + j, 0), kmi = C(o.G, ng, 6 + i, 6 + r + j, 1);
        const double mkr = C(o.G, ng, 6 + r + i, 6 + j, 0), mki = C(o.G, ng, 6 + r + i, 6 + j, 1);
        dst[L.J + 2 * ((size_t)i * R + j)] = -(kmi - mki);
        dst[L.J + 2 * ((size_t)i * R + j) + 1] = kmr - mkr;
      }
    }
  for (int c3 = 0; c3 < 3; ++c3)
    for (int i = 0; i < r; ++i)
      for (int c = 0; c < 2; ++c) {
        dst[L.b0 + 2 * ((size_t)c3 * R + i) + c] = o.b0[2 * ((size_t)i * 3 + c3) + c];
        dst[L.b1 + 2 * ((size_t)c3 * R + i) + c] = o.b1[2 * ((size_t)i * 3 + c3) + c];
        dst[L.H + 2 * ((size_t)c3 * R + i) + c] = o.H[2 * ((size_t)c3 * r + i) + c];
      }
  for (int a = 0; a < 6; ++a) {
    for (int i = 0; i < r; ++i)
      for (int c = 0; c < 2; ++c) {
        dst[L.GbK + 2 * ((size_t)a * R + i) + c] = C(o.G, ng, a, 6 + i, c);
        dst[L.GbM + 2 * ((size_t)a * R + i) + c] = C(o.G, ng, a, 6 + r + i, c);
      }
    for (int b = 0; b < 6; ++b)
      for (int c = 0; c < 2; ++c) dst[L.Gbb + 2 * (a * 6 + b) + c] = C(o.G, ng, a, b, c);
  }
  double *sc = dst + L.scal;
  sc[podp::SC_NU] = o.nu;
  sc[podp::SC_PENCIL_OK] = 0.0;
  sc[podp::SC_ALPHA] = o.alpha;
  sc[podp::SC_ALPHA_LB] = o.alpha_lb;
  for (int e = 0; e < 9; ++e) {
    sc[podp::SC_S + e] = o.S[e];
    sc[podp::SC_N0 + e] = o.N0[e];
  }
}

// One stream-ordered memory pool per device for the whole library (P hand-off workspaces, LU scratch, select
// scratch), created on first use and kept for the process: its release threshold is infinite, so steady-state
// evaluations -- across contexts too, e.g. the one context per iteration of the Algorithm-1 driver -- reuse mapped
// memory instead of paying for a fresh pool and fresh mappings per context.
std::mutex g_pool_mu;
std::vector<cudaMemPool_t> g_pools;

cudaError_t library_pool(int device, cudaMemPool_t *out) {
  std::mutex &mu = g_pool_mu;
  std::vector<cudaMemPool_t> &pools = g_pools;
  std::lock_guard<std::mutex> lk(mu);
  if ((int)pools.size() <= device) pools.resize(device + 1, nullptr);
  if (!pools[device]) {
    cudaMemPoolProps pp = {};
    pp.allocType = cudaMemAllocationTypePinned;
    pp.handleTypes = cudaMemHandleTypeNone;
    pp.location.type = cudaMemLocationTypeDevice;
    pp.location.id = device;
    cudaMemPool_t pool = nullptr;
    cudaError_t e = cudaMemPoolCreate(&pool, &pp);
    if (e != cudaSuccess) return e;
    uint64_t thr = UINT64_MAX;  // never trim
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    pools[device] = pool;
  }
  *out = pools[device];
  return cudaSuccess;
}

// Padded size: next multiple of 8 (the specialised kernels exist for R = 8, 16, ..., 128); the padding is exact
// (K_pad = diag(K, I), every other operator zero-padded).
int choose_R(int r) { return (r + 7) / 8 * 8; }

// N3 precompute for every object (Cholesky, Jacobi, Z, c0, c1 on the true r; the padding extends it exactly with
// Z_pad = diag(Z, I), lambda_pad = 0, c_pad = 0), then the operators in pencil coordinates; uploads only the
// pencil blocks.  Called once, under ctx->pencil_mu, by the first PODP_FLAG_PENCIL evaluation.
podp_status pencil_prepare(podp_ctx *c, cudaStream_t s) {
  const podp::Layout &L = c->L;
  const int r = c->r, R = L.R;
  std::vector<double> host((size_t)L.stride * c->n_obj, 0.0);
  cudaError_t e = cudaMemcpyAsync(host.data(), c->d_ops, host.size() * sizeof(double), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "pencil precompute: download operators");
  bool ok = true, diag = true;
  for (int k = 0; k < c->n_obj; ++k) {
    double *dst = host.data() + (size_t)L.stride * k;
    std::vector<double> Z, lam, c0, c1;
    const size_t rr = (size_t)2 * r * r, r3 = (size_t)6 * r;
    if (!podp::pencil_precompute(r, c->hK.data() + rr * k, c->hM.data() + rr * k, c->hb0.data() + r3 * k,
                                 c->hb1.data() + r3 * k, Z, lam, c0, c1)) {
      ok = false;
      break;
    }
    for (int i = 0; i < R; ++i)
      for (int j = 0; j < R; ++j) {
        const size_t el = 2 * ((size_t)i * R + j);
        const bool in = i < r && j < r;
        dst[L.Z + el] = in ? Z[2 * ((size_t)i * r + j)] : (i == j ? 1.0 : 0.0);
        dst[L.Z + el + 1] = in ? Z[2 * ((size_t)i * r + j) + 1] : 0.0;
      }
    for (int el = 0; el < r; ++el) dst[L.lam + el] = lam[el];
    for (int c3 = 0; c3 < 3; ++c3)
      for (int kk = 0; kk < r; ++kk)
        for (int cc = 0; cc < 2; ++cc) {
          dst[L.c0 + 2 * ((size_t)c3 * R + kk) + cc] = c0[2 * ((size_t)c3 * r + kk) + cc];
          dst[L.c1 + 2 * ((size_t)c3 * R + kk) + cc] = c1[2 * ((size_t)c3 * r + kk) + cc];
        }
    pencil_transform(L, dst);
    diag &= !c->has_KR_MI[k];
  }
  c->pencil_done = true;
  c->pencil_ok = ok;
  c->pencil_diag = ok && diag;
  if (!ok) return PODP_OK;
  // the pencil blocks are contiguous from L.Z to the end of each object's stride
  for (int k = 0; k < c->n_obj && e == cudaSuccess; ++k) {
    const size_t off = (size_t)L.stride * k + L.Z;
    e = cudaMemcpyAsync(c->d_ops + off, host.data() + off, sizeof(double) * (L.stride - L.Z), cudaMemcpyHostToDevice, s);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    c->pencil_ok = false;
    return cuda_fail(e, "pencil precompute: upload");
  }
  return PODP_OK;
}

}  // namespace

namespace podp {
Layout make_layout(int R) {
  Layout L;
  L.R = R;
  int64_t off = 0;
  auto take = [&](int64_t n) {
    int64_t o = off;
    off += (n + 31) / 32 * 32;  // 256-byte aligned blocks
    return o;
  };
  const int64_t sq = 2LL * R * R, vec3 = 6LL * R, vec6 = 12LL * R;
  L.K = take(sq);
  L.M = take(sq);
  L.KR = take(sq);
  L.MI = take(sq);
  L.Gkk = take(sq);
  L.J = take(sq);
  L.Gmm = take(sq);
  L.b0 = take(vec3);
  L.b1 = take(vec3);
  L.H = take(vec3);
  L.GbK = take(vec6);
  L.GbM = take(vec6);
  L.Gbb = take(72);
  L.scal = take(SCAL_N);
  L.Z = take(sq);
  L.lam = take(R);
  L.c0 = take(vec3);
  L.c1 = take(vec3);
  L.PKR = take(sq);
  L.PMI = take(sq);
  L.PGkk = take(sq);
  L.PJ = take(sq);
  L.PGmm = take(sq);
  L.PH = take(vec3);
  L.PGbK = take(vec6);
  L.PGbM = take(vec6);
  L.stride = off;
  return L;
}
}  // namespace podp

extern "C" {

const char *podp_last_error(void) { return g_err.c_str(); }

podp_status podp_release_workspace(int device) {
  g_err.clear();
  std::lock_guard<std::mutex> lk(g_pool_mu);
  if (device < 0 || device >= (int)g_pools.size() || !g_pools[device])
    return fail(PODP_ERR_ARG, "no workspace pool on device %d", device);
  cudaError_t e = cudaMemPoolTrimTo(g_pools[device], 0);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemPoolTrimTo");
  return PODP_OK;
}
const char *podp_version(void) { return "podp-b200 0.1 (sm_100a, fp64)"; }
int32_t podp_last_launch_count(void) { return g_last_launches; }
int32_t podp_n_obj(const podp_ctx *c) { return c ? c->n_obj : 0; }
int32_t podp_r(const podp_ctx *c) { return c ? c->r : 0; }

podp_status podp_create_batch(int32_t n_obj, const podp_operators *ops, int device, void *cuda_stream,
                              podp_ctx **out) {
  g_err.clear();
  if (!out) return fail(PODP_ERR_ARG, "out is NULL");
  *out = nullptr;
  if (n_obj < 1 || !ops) return fail(PODP_ERR_ARG, "n_obj must be >= 1 and ops non-NULL");
  for (int k = 0; k < n_obj; ++k) {
    podp_status st = validate(ops[k], k);
    if (st != PODP_OK) return st;
    if (ops[k].r != ops[0].r) return fail(PODP_ERR_ARG, "object %d: r=%d differs from object 0 (r=%d)", k, ops[k].r, ops[0].r);
  }
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
  if (device < 0 || device >= ndev) return fail(PODP_ERR_ARG, "device %d out of range (%d devices)", device, ndev);
  int cc_major = 0, cc_minor = 0;  // (attribute queries: cudaGetDeviceProperties costs milliseconds)
  e = cudaDeviceGetAttribute(&cc_major, cudaDevAttrComputeCapabilityMajor, device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&cc_minor, cudaDevAttrComputeCapabilityMinor, device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
  if (cc_major != 10) return fail(PODP_ERR_UNSUPPORTED, "device %d is sm_%d%d; libpodp is built for sm_100a", device, cc_major, cc_minor);
  DeviceGuard guard(device);
  if (!guard.ok) return fail(PODP_ERR_CUDA, "cudaSetDevice(%d) failed", device);
  const int r = ops[0].r;
  podp::Layout L = podp::make_layout(choose_R(r));
  std::vector<double> host((size_t)L.stride * n_obj, 0.0);
  for (int k = 0; k < n_obj; ++k) pack(ops[k], L, host.data() + (size_t)L.stride * k);
  cudaMemPool_t pool = nullptr;
  e = library_pool(device, &pool);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemPoolCreate");
  // the packed operators come from the library pool too (no cudaMalloc / cudaFree, which synchronise the device)
  double *d = nullptr;
  cudaStream_t s = (cudaStream_t)cuda_stream;
  e = cudaMallocFromPoolAsync((void **)&d, host.size() * sizeof(double), pool, s);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync(operators)");
  e = cudaMemcpyAsync(d, host.data(), host.size() * sizeof(double), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    cudaFreeAsync(d, s);
    return cuda_fail(e, "upload operators");
  }
  podp_ctx *c = new podp_ctx;
  {
    const size_t rr = (size_t)2 * r * r, r3 = (size_t)6 * r;
    c->hK.resize(rr * n_obj);
    c->hM.resize(rr * n_obj);
    c->hb0.resize(r3 * n_obj);
    c->hb1.resize(r3 * n_obj);
    c->has_KR_MI.resize(n_obj);
    for (int k = 0; k < n_obj; ++k) {
      std::memcpy(c->hK.data() + rr * k, ops[k].K, rr * sizeof(double));
      std::memcpy(c->hM.data() + rr * k, ops[k].M, rr * sizeof(double));
      std::memcpy(c->hb0.data() + r3 * k, ops[k].b0, r3 * sizeof(double));
      std::memcpy(c->hb1.data() + r3 * k, ops[k].b1, r3 * sizeof(double));
      c->has_KR_MI[k] = ops[k].K_R != nullptr || ops[k].M_I != nullptr;
    }
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  c->sms = sms;
  c->pool = pool;
  c->device = device;
  c->r = r;
  c->n_obj = n_obj;
  c->L = L;
  c->d_ops = d;
  *out = c;
  return PODP_OK;
}

podp_status podp_create(const podp_operators *ops, int device, void *cuda_stream, podp_ctx **out) {
  return podp_create_batch(1, ops, device, cuda_stream, out);
}

podp_status podp_invariants(const double *T1_d, const double *I_d, int64_t n, double *eigR_d, double *eigI_d,
                            void *cuda_stream) {
  g_err.clear();
  if (n < 0) return fail(PODP_ERR_ARG, "n < 0");
  if (n == 0) return PODP_OK;
  if (!T1_d || !I_d || !eigR_d || !eigI_d) return fail(PODP_ERR_ARG, "null pointer");
  cudaError_t e = podp::launch_invariants(T1_d, I_d, n, eigR_d, eigI_d, (cudaStream_t)cuda_stream);
  if (e != cudaSuccess) return cuda_fail(e, "podp_invariants");
  return PODP_OK;
}

podp_status podp_coil_voltage(const double *T1_d, const double *I_d, int64_t n, const double *h_ex,
                              const double *h_ms, int32_t n_coil, double *V_d, void *cuda_stream) {
  g_err.clear();
  if (n < 0) return fail(PODP_ERR_ARG, "n < 0");
  if (n_coil < 1 || n_coil > 64) return fail(PODP_ERR_ARG, "need 1 <= n_coil <= 64");
  if (!h_ex || !h_ms) return fail(PODP_ERR_ARG, "null coil field pointer");
  if (n == 0) return PODP_OK;
  if (!T1_d || !I_d || !V_d) return fail(PODP_ERR_ARG, "null pointer");
  cudaStream_t s = (cudaStream_t)cuda_stream;
  double *h = nullptr;
  cudaError_t e = cudaMallocAsync((void **)&h, sizeof(double) * 6 * n_coil, s);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync(coil fields)");
  e = cudaMemcpyAsync(h, h_ex, sizeof(double) * 3 * n_coil, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(h + 3 * n_coil, h_ms, sizeof(double) * 3 * n_coil, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = podp::launch_coil_voltage(T1_d, I_d, n, h, h + 3 * n_coil, n_coil, V_d, s);
  cudaFreeAsync(h, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // host arrays may be released by the caller
  if (e != cudaSuccess) return cuda_fail(e, "podp_coil_voltage");
  return PODP_OK;
}

podp_status podp_profile_enable(int on) {
  g_prof_on = on != 0;
  return PODP_OK;
}

int32_t podp_profile_read(char *names, double *ms, int64_t *counts, int32_t max_entries, int32_t reset) {
  for (auto &pp : g_prof_pending) {
    float t = 0.f;
    cudaEventSynchronize(pp.b);
    cudaEventElapsedTime(&t, pp.a, pp.b);
    cudaEventDestroy(pp.a);
    cudaEventDestroy(pp.b);
    bool found = false;
    for (auto &acc : g_prof_acc)
      if (acc.first == pp.name) {
        acc.second.first += t;
        acc.second.second += 1;
        found = true;
      }
    if (!found) g_prof_acc.push_back({pp.name, {t, 1}});
  }
  g_prof_pending.clear();
  int32_t n = 0;
  for (auto &acc : g_prof_acc) {
    if (n >= max_entries) break;
    if (names) {
      strncpy(names + 32 * n, acc.first.c_str(), 31);
      names[32 * n + 31] = 0;
    }
    if (ms) ms[n] = acc.second.first;
    if (counts) counts[n] = acc.second.second;
    ++n;
  }
  if (reset) g_prof_acc.clear();
  return n;
}

podp_status podp_destroy(podp_ctx *c) {
  if (!c) return PODP_OK;
  for (int i = 0; i < 3; ++i)
    if (c->dir[i]) podp_destroy(c->dir[i]);
  DeviceGuard guard(c->device);
  cudaDeviceSynchronize();
  // every stream's work on the context is complete after the device synchronisation; the operators go back to the
  // library pool (shared by every context on the device)
  cudaFreeAsync(c->d_ops, 0);
  if (c->copy_stream) {
    cudaStreamDestroy(c->copy_stream);
    cudaEventDestroy(c->ev_half);
    cudaEventDestroy(c->ev_copied);
  }
  delete c;
  return PODP_OK;
}

}  // extern "C"

namespace {

enum SolverKind { K_LL, K_BLK, K_DYN, K_GEN, K_PENCIL };

// Solver for padded size R: the one-warp left-looking kernel up to R = 96 (pivoting or PODP_FLAG_NO_PIVOT), the
// generic kernel beyond; PODP_FLAG_LU_* overrides (A/B: the lock-step and dynamically scheduled blocked kernels).
podp_status pick_solver(int R, int flags, SolverKind *ker) {
  const int lu_sel = flags & (PODP_FLAG_LU_LL | PODP_FLAG_LU_BLK | PODP_FLAG_LU_DYN | PODP_FLAG_LU_GENERIC);
  if (lu_sel & (lu_sel - 1)) return fail(PODP_ERR_ARG, "at most one PODP_FLAG_LU_* solver may be requested");
  if ((lu_sel == PODP_FLAG_LU_LL && R > 96) || ((lu_sel == PODP_FLAG_LU_BLK || lu_sel == PODP_FLAG_LU_DYN) && R > 96))
    return fail(PODP_ERR_UNSUPPORTED, "requested LU kernel is not instantiated for padded r = %d", R);
  if ((lu_sel == PODP_FLAG_LU_BLK || lu_sel == PODP_FLAG_LU_DYN) && (flags & PODP_FLAG_NO_PIVOT))
    return fail(PODP_ERR_UNSUPPORTED, "PODP_FLAG_LU_BLK / _DYN always pivot");
  if (flags & PODP_FLAG_PENCIL) *ker = K_PENCIL;
  else if (lu_sel == PODP_FLAG_LU_LL) *ker = K_LL;
  else if (lu_sel == PODP_FLAG_LU_BLK) *ker = K_BLK;
  else if (lu_sel == PODP_FLAG_LU_DYN) *ker = K_DYN;
  else if (lu_sel == PODP_FLAG_LU_GENERIC) *ker = K_GEN;
  else if (R <= 96) *ker = K_LL;  // measured fastest at every padded R = 8 .. 96 (profiles/r02_luab_layout.txt)
  else *ker = K_GEN;
  return PODP_OK;
}

size_t solver_scratch_bytes(SolverKind ker, int R, int sms) {
  if (ker == K_LL) return podp::lu_ll_scratch_bytes(R, sms);
  if (ker == K_DYN) return podp::lu_dyn_scratch_bytes(R, sms);
  if (ker == K_GEN) return podp::solve_scratch_bytes(R, sms);
  return 0;
}

cudaError_t launch_solver(SolverKind ker, const podp::EvalArgs &a, cudaStream_t s, int sms, bool pencil_y) {
  switch (ker) {
    case K_PENCIL: return pencil_y ? podp::launch_pencil_y(a, s) : podp::launch_pencil(a, s);
    case K_LL: return podp::launch_lu_ll(a, s, sms);
    case K_BLK: return podp::launch_lu_blk(a, s);
    case K_DYN: return podp::launch_lu_dyn(a, s);
    case K_GEN: return podp::launch_solve(a, s, a.gscr);
  }
  return cudaErrorInvalidValue;
}

podp::EvalArgs make_args(const podp_ctx *c, const double *omega_d, int64_t F, double *T1_d, double *I_d,
                         double *Delta_d, int32_t *info_d, double *P_out, int flags) {
  podp::EvalArgs a;
  a.ops = c->d_ops;
  a.L = c->L;
  a.r = c->r;
  a.n_obj = c->n_obj;
  a.omega = omega_d;
  a.F = F;
  a.T1 = T1_d;
  a.I = I_d;
  a.Delta = Delta_d;
  a.info = info_d;
  a.P_out = P_out;
  a.flags = flags;
  a.Pws = nullptr;
  a.gscr = nullptr;
  a.blk_hi[0] = a.blk_hi[1] = 0;
  return a;
}

// N1 literal form: three direction solves (batch of 3 objects of padded size R_s) -> placement into the
// concatenated columns -> the contraction kernel with the cross-block operators of this context.
podp_status eval_perdir(podp_ctx *c, const double *omega_d, int64_t F, double *T1_d, double *I_d, double *Delta_d,
                        int32_t *info_d, double *P_d, int flags, cudaStream_t s) {
  if (flags & PODP_FLAG_PENCIL) return fail(PODP_ERR_UNSUPPORTED, "PODP_FLAG_PENCIL on a per-direction context");
  const int Re = c->L.R;
  SolverKind ker[3];
  int Rs[3];
  size_t p3[3], gsz[3], total = 0;
  for (int i = 0; i < 3; ++i) {
    Rs[i] = c->dir[i]->L.R;
    podp_status st = pick_solver(Rs[i], flags, &ker[i]);
    if (st != PODP_OK) return st;
    p3[i] = (size_t)F * 3 * Rs[i] * sizeof(double2);
    gsz[i] = (solver_scratch_bytes(ker[i], Rs[i], c->sms) + 255) / 256 * 256;
    total += p3[i] + gsz[i];
  }
  const size_t pe = (size_t)F * 3 * Re * sizeof(double2);
  const size_t in3 = (((size_t)3 * F * sizeof(int32_t)) + 255) / 256 * 256;
  char *buf = nullptr;
  cudaError_t e = cudaMallocFromPoolAsync((void **)&buf, total + pe + in3, c->pool, s);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync(per-direction workspace)");
  double2 *Pe = reinterpret_cast<double2 *>(buf);
  int32_t *info3 = reinterpret_cast<int32_t *>(buf + pe);
  const double2 *Pd[3];
  int nl = 0;
  size_t at = pe + in3;
  for (int i = 0; i < 3 && e == cudaSuccess; ++i) {
    podp::EvalArgs ai = make_args(c->dir[i], omega_d, F, nullptr, nullptr, nullptr, info3 + (size_t)i * F, nullptr,
                                  flags & ~(PODP_FLAG_OUT_P));
    ai.Pws = reinterpret_cast<double2 *>(buf + at);
    Pd[i] = ai.Pws;
    at += p3[i];
    ai.gscr = gsz[i] ? reinterpret_cast<double2 *>(buf + at) : nullptr;
    at += gsz[i];
    ProfScope ps("solve", s);
    e = launch_solver(ker[i], ai, s, c->sms, false);
    if (e == cudaSuccess) ++nl;
  }
  if (e == cudaSuccess) {
    ProfScope ps("scatter", s);
    e = podp::launch_perdir_scatter(Pd, Rs, c->m, c->offp, info3, F, Pe, Re, info_d,
                                    (flags & PODP_FLAG_OUT_P) ? P_d : nullptr, s);
    if (e == cudaSuccess) ++nl;
  }
  if (e == cudaSuccess) {
    podp::EvalArgs am = make_args(c, omega_d, F, T1_d, I_d, Delta_d, nullptr, nullptr, flags);
    am.Pws = Pe;
    am.blk_hi[0] = c->offp[1];
    am.blk_hi[1] = c->offp[2];
    ProfScope ps("mpt", s);
    e = podp::launch_mpt_tile(am, s, false);
    if (e == cudaSuccess) ++nl;
  }
  cudaFreeAsync(buf, s);
  g_last_launches = nl;
  if (e != cudaSuccess) return cuda_fail(e, "podp_eval (per-direction) launch");
  return PODP_OK;
}

}  // namespace

extern "C" {

podp_status podp_eval(const podp_ctx *cc, const double *omega_d, int64_t F, double *T1_d, double *I_d,
                      double *Delta_d, int32_t *info_d, double *P_d, int flags, void *cuda_stream) {
  g_err.clear();
  g_last_launches = 0;
  podp_ctx *c = const_cast<podp_ctx *>(cc);  // only the lazily built pencil precompute is ever written
  if (!c) return fail(PODP_ERR_ARG, "ctx is NULL");
  if (F < 0) return fail(PODP_ERR_ARG, "F < 0");
  if (F == 0) return PODP_OK;
  if (!omega_d || !T1_d || !I_d || !Delta_d) return fail(PODP_ERR_ARG, "null omega/output pointer");
  if ((flags & PODP_FLAG_OUT_P) && !P_d) return fail(PODP_ERR_ARG, "PODP_FLAG_OUT_P set but P_d is NULL");
  const int known = PODP_FLAG_OUT_R | PODP_FLAG_OUT_P | PODP_FLAG_NO_PIVOT | PODP_FLAG_PENCIL | PODP_FLAG_LU_LL |
                    PODP_FLAG_LU_BLK | PODP_FLAG_LU_DYN | PODP_FLAG_LU_GENERIC | PODP_FLAG_MPT_GEMM |
                    PODP_FLAG_MPT_PAIR;
  if (flags & ~known) return fail(PODP_ERR_ARG, "unknown flag bits 0x%x", flags & ~known);
  DeviceGuard guard(c->device);
  if (!guard.ok) return fail(PODP_ERR_CUDA, "cudaSetDevice(%d) failed", c->device);
  cudaStream_t s = (cudaStream_t)cuda_stream;
  if (c->dir[0]) return eval_perdir(c, omega_d, F, T1_d, I_d, Delta_d, info_d, P_d, flags, s);
  const int R = c->L.R;
  SolverKind ker;
  podp_status st0 = pick_solver(R, flags, &ker);
  if (st0 != PODP_OK) return st0;
  if ((flags & PODP_FLAG_MPT_PAIR) && (c->n_obj != 1 || (flags & (PODP_FLAG_PENCIL | PODP_FLAG_MPT_GEMM)) || R != 48))
    return fail(PODP_ERR_UNSUPPORTED, "PODP_FLAG_MPT_PAIR: one object, padded r = 48, no pencil");
  if ((flags & PODP_FLAG_MPT_GEMM) && (c->n_obj != 1 || (flags & PODP_FLAG_PENCIL) || !(R == 24 || R == 48 || R == 96)))
    return fail(PODP_ERR_UNSUPPORTED, "PODP_FLAG_MPT_GEMM: one object, padded r in {24, 48, 96}, no pencil");
  if (flags & PODP_FLAG_PENCIL) {
    std::lock_guard<std::mutex> lk(c->pencil_mu);
    if (!c->pencil_done) {
      podp_status st = pencil_prepare(c, s);
      if (st != PODP_OK) return st;
    }
    if (!c->pencil_ok)
      return fail(PODP_ERR_UNSUPPORTED, "PODP_FLAG_PENCIL needs K Hermitian positive definite (Cholesky failed)");
  }
  podp::EvalArgs a = make_args(c, omega_d, F, T1_d, I_d, Delta_d, info_d,
                               (flags & PODP_FLAG_OUT_P) ? P_d : nullptr, flags);
  const size_t gsz = solver_scratch_bytes(ker, R, c->sms);
  const size_t ws = (size_t)c->n_obj * (size_t)F * 3 * R * sizeof(double2);
  cudaError_t e = cudaMallocFromPoolAsync((void **)&a.Pws, ws, c->pool, s);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync(P workspace)");
  if (gsz) {
    e = cudaMallocFromPoolAsync((void **)&a.gscr, gsz, c->pool, s);
    if (e != cudaSuccess) {
      cudaFreeAsync(a.Pws, s);
      return cuda_fail(e, "cudaMallocAsync(LU scratch)");
    }
  }
  int nl = 0;
  // N3 without the debug P output: solve for y only and run the MPT/certificate kernel in pencil coordinates
  const bool pencil_y = (flags & PODP_FLAG_PENCIL) && !(flags & PODP_FLAG_OUT_P);
  podp::EvalArgs am = a;
  if (pencil_y) {
    am.L.KR = c->L.PKR;
    am.L.MI = c->L.PMI;
    am.L.Gkk = c->L.PGkk;
    am.L.J = c->L.PJ;
    am.L.Gmm = c->L.PGmm;
    am.L.H = c->L.PH;
    am.L.GbK = c->L.PGbK;
    am.L.GbM = c->L.PGbM;
  }
  {
    ProfScope ps("solve", s);
    e = launch_solver(ker, a, s, c->sms, pencil_y);
    if (e == cudaSuccess) ++nl;
  }
  if (e == cudaSuccess) {
    ProfScope ps("mpt", s);
    HostSplit *hs = g_split;
    if (hs && c->n_obj == 1 && !(flags & PODP_FLAG_MPT_GEMM) && F >= 2 * HOST_SPLIT_MIN) {
      // two launches over the halves (whole contraction tiles: no extra tail), first half's rows copied meanwhile
      const int64_t F1 = (F / 2) / 64 * 64;
      podp::EvalArgs a1 = am, a2 = am;
      a1.F = F1;
      a2.F = F - F1;
      a2.omega += F1;
      a2.Pws += (size_t)F1 * 3 * R;
      a2.T1 += F1 * 6;
      a2.I += F1 * 6;
      a2.Delta += F1 * 6;
      e = podp::launch_mpt_tile(a1, s, pencil_y && c->pencil_diag);
      if (e == cudaSuccess) e = cudaEventRecord(hs->ev, s);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(hs->cs, hs->ev, 0);
      const size_t nb = sizeof(double) * (size_t)F1 * 6;
      if (e == cudaSuccess) e = cudaMemcpyAsync(hs->T1_h, am.T1, nb, cudaMemcpyDeviceToHost, hs->cs);
      if (e == cudaSuccess) e = cudaMemcpyAsync(hs->I_h, am.I, nb, cudaMemcpyDeviceToHost, hs->cs);
      if (e == cudaSuccess) e = cudaMemcpyAsync(hs->D_h, am.Delta, nb, cudaMemcpyDeviceToHost, hs->cs);
      if (e == cudaSuccess) {
        ++nl;
        hs->F1 = F1;
        e = podp::launch_mpt_tile(a2, s, pencil_y && c->pencil_diag);
      }
    } else {
      e = (flags & PODP_FLAG_MPT_GEMM) ? podp::launch_mpt_gemm(am, s, c->sms)
                                       : podp::launch_mpt_tile(am, s, pencil_y && c->pencil_diag);
    }
    if (e == cudaSuccess) ++nl;
  }
  cudaFreeAsync(a.Pws, s);
  if (a.gscr) cudaFreeAsync(a.gscr, s);
  g_last_launches = nl;
  if (e != cudaSuccess) return cuda_fail(e, "podp_eval launch");
  return PODP_OK;
}

podp_status podp_eval_host(const podp_ctx *c, const double *omega_h, int64_t F, double *T1_h, double *I_h,
                           double *Delta_h, int32_t *info_h, int flags, void *cuda_stream) {
  g_err.clear();
  if (!c) return fail(PODP_ERR_ARG, "ctx is NULL");
  if (F < 0) return fail(PODP_ERR_ARG, "F < 0");
  if (F == 0) return PODP_OK;
  if (!omega_h || !T1_h || !I_h || !Delta_h) return fail(PODP_ERR_ARG, "null omega/output pointer");
  if (flags & PODP_FLAG_OUT_P) return fail(PODP_ERR_ARG, "PODP_FLAG_OUT_P is not available on the host entry point");
  DeviceGuard guard(c->device);
  if (!guard.ok) return fail(PODP_ERR_CUDA, "cudaSetDevice(%d) failed", c->device);
  cudaStream_t s = (cudaStream_t)cuda_stream;
  const size_t nout = (size_t)c->n_obj * F * 6;
  auto up = [](size_t b) { return (b + 255) / 256 * 256; };  // 256-byte aligned sub-buffers (vector stores)
  const size_t b_om = up(sizeof(double) * F), b_out = up(sizeof(double) * nout);
  const size_t bytes = b_om + 3 * b_out + sizeof(int32_t) * (size_t)c->n_obj * F;
  char *buf = nullptr;
  cudaError_t e = cudaMallocFromPoolAsync((void **)&buf, bytes, c->pool, s);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync(host eval staging)");
  double *om = (double *)buf, *T1 = (double *)(buf + b_om), *I = (double *)(buf + b_om + b_out),
         *D = (double *)(buf + b_om + 2 * b_out);
  int32_t *info = (int32_t *)(buf + b_om + 3 * b_out);
  e = cudaMemcpyAsync(om, omega_h, sizeof(double) * F, cudaMemcpyHostToDevice, s);
  podp_status st = PODP_OK;
  bool split_used = false;
  podp_ctx *cw = const_cast<podp_ctx *>(c);
  // host evaluations of one context share its copy stream and events: they are serialised (they would share the GPU
  // anyway); device-pointer evaluations (podp_eval) stay fully concurrent
  std::lock_guard<std::mutex> host_lk(cw->host_mu);
  if (e == cudaSuccess) {
    // the first half of the outputs is copied back on the context's copy stream while the contraction kernel works
    // on the second half (podp_eval, HostSplit)
    HostSplit hs{T1_h, I_h, Delta_h, nullptr, nullptr, 0};
    {
      if (!cw->copy_stream) {
        if (cudaStreamCreateWithFlags(&cw->copy_stream, cudaStreamNonBlocking) != cudaSuccess) cw->copy_stream = nullptr;
        if (cw->copy_stream && (cudaEventCreateWithFlags(&cw->ev_half, cudaEventDisableTiming) != cudaSuccess ||
                                cudaEventCreateWithFlags(&cw->ev_copied, cudaEventDisableTiming) != cudaSuccess)) {
          cudaStreamDestroy(cw->copy_stream);
          cw->copy_stream = nullptr;
        }
      }
      hs.cs = cw->copy_stream;
      hs.ev = cw->ev_half;
    }
    g_split = hs.cs ? &hs : nullptr;
    st = podp_eval(c, om, F, T1, I, D, info_h ? info : nullptr, nullptr, flags, s);
    g_split = nullptr;
    const int64_t F1 = hs.F1;  // frequencies already on their way to the host (one object)
    split_used = F1 > 0;
    if (st == PODP_OK) {
      const size_t off = (size_t)F1 * 6, nb = sizeof(double) * (nout - off);
      e = cudaMemcpyAsync(T1_h + off, T1 + off, nb, cudaMemcpyDeviceToHost, s);
      if (e == cudaSuccess) e = cudaMemcpyAsync(I_h + off, I + off, nb, cudaMemcpyDeviceToHost, s);
      if (e == cudaSuccess) e = cudaMemcpyAsync(Delta_h + off, D + off, nb, cudaMemcpyDeviceToHost, s);
      if (e == cudaSuccess && info_h)
        e = cudaMemcpyAsync(info_h, info, sizeof(int32_t) * c->n_obj * F, cudaMemcpyDeviceToHost, s);
    }
    if (split_used) {  // the staging buffer is released (stream-ordered on s) only after the copy stream is done
      cudaEventRecord(cw->ev_copied, cw->copy_stream);
      cudaStreamWaitEvent(s, cw->ev_copied, 0);
    }
  }
  cudaFreeAsync(buf, s);
  cudaError_t e2 = cudaStreamSynchronize(s);
  if (st != PODP_OK) return st;
  if (e != cudaSuccess) return cuda_fail(e, "podp_eval_host copies");
  if (e2 != cudaSuccess) return cuda_fail(e2, "podp_eval_host synchronize");
  return PODP_OK;
}

podp_status podp_select(const podp_ctx *c, const double *omega_d, const double *Delta_d, int64_t F,
                        const double *snap, int32_t n_snap, int32_t n_star, double theta, int32_t *n_new,
                        double *omega_new, int64_t *idx_new, double *Lambda, double *Lambda_n, void *cuda_stream) {
  g_err.clear();
  g_last_launches = 0;
  if (!c) return fail(PODP_ERR_ARG, "ctx is NULL");
  if (F < 0 || (F > 0 && (!omega_d || !Delta_d))) return fail(PODP_ERR_ARG, "bad omega/Delta/F");
  if (!snap || n_snap < 2 || n_snap > PODP_SNAP_MAX) return fail(PODP_ERR_ARG, "need 2 <= n_snap <= %d", PODP_SNAP_MAX);
  for (int i = 0; i < n_snap; ++i) {
    if (!std::isfinite(snap[i])) return fail(PODP_ERR_ARG, "snapshot %d is not finite", i);
    if (i && !(snap[i] > snap[i - 1])) return fail(PODP_ERR_ARG, "snapshots must be strictly ascending");
  }
  if (n_star < 1 || n_star > 64) return fail(PODP_ERR_ARG, "need 1 <= n_star <= 64");
  if (!(theta <= 1.0) || std::isnan(theta)) return fail(PODP_ERR_ARG, "theta must be <= 1 (<= 0 selects top-N* mode)");
  if (!n_new || !omega_new || !idx_new || !Lambda) return fail(PODP_ERR_ARG, "null output pointer");
  DeviceGuard guard(c->device);
  if (!guard.ok) return fail(PODP_ERR_CUDA, "cudaSetDevice(%d) failed", c->device);
  cudaStream_t s = (cudaStream_t)cuda_stream;
  const int n_int = n_snap - 1;
  const size_t n_res = 2 + n_int + 2 * (size_t)n_star;
  const size_t bytes = sizeof(double) * (n_snap + n_res) + 2 * sizeof(unsigned long long) * n_int;
  char *buf = nullptr;
  cudaError_t e = cudaMallocFromPoolAsync((void **)&buf, bytes, c->pool, s);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync(select scratch)");
  double *snap_d = (double *)buf, *res_d = snap_d + n_snap;
  unsigned long long *keys = (unsigned long long *)(res_d + n_res), *args = keys + n_int;
  std::vector<double> res(n_res);
  int nl = 0;
  e = cudaMemcpyAsync(snap_d, snap, sizeof(double) * n_snap, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) {
    ProfScope ps("select", s);
    e = podp::launch_select(omega_d, Delta_d, F, snap_d, n_snap, n_star, theta, keys, args, res_d, s, &nl);
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(res.data(), res_d, sizeof(double) * n_res, cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(buf, s);
  cudaError_t e2 = cudaStreamSynchronize(s);
  g_last_launches = nl;
  if (e != cudaSuccess) return cuda_fail(e, "podp_select");
  if (e2 != cudaSuccess) return cuda_fail(e2, "podp_select synchronize");
  if (Lambda_n)
    for (int n = 0; n < n_int; ++n) Lambda_n[n] = res[2 + n];
  *Lambda = res[1];
  const int nc = (int)res[0];
  if (nc < 0) {
    *n_new = 0;
    return fail(PODP_ERR_NO_CANDIDATES, "fewer non-empty intervals than requested");
  }
  *n_new = nc;
  for (int q = 0; q < n_star; ++q) {
    idx_new[q] = q < nc ? (int64_t)res[2 + n_int + q] : -1;
    omega_new[q] = q < nc ? res[2 + n_int + n_star + q] : std::nan("");
  }
  return PODP_OK;
}

podp_status podp_create_perdir(const podp_perdir_operators *o, int device, void *cuda_stream, podp_ctx **out) {
  g_err.clear();
  if (!out) return fail(PODP_ERR_ARG, "out is NULL");
  *out = nullptr;
  if (!o) return fail(PODP_ERR_ARG, "ops is NULL");
  int off[4] = {0, 0, 0, 0};
  for (int i = 0; i < 3; ++i) {
    if (o->m[i] < 1) return fail(PODP_ERR_ARG, "M_%d = %d must be >= 1", i + 1, o->m[i]);
    off[i + 1] = off[i] + o->m[i];
  }
  if (off[3] > PODP_R_MAX) return fail(PODP_ERR_ARG, "M_1 + M_2 + M_3 = %d exceeds %d", off[3], PODP_R_MAX);
  // concatenation with each direction block padded to the contraction kernel's b-slice width (8 up to 64 rows,
  // else 16), so the kernel can skip the zero blocks per b-group; the padding rows and columns are exact zeros
  int pad = 8, offp[4] = {0, 0, 0, 0};
  for (int pass = 0; pass < 2; ++pass) {
    for (int i = 0; i < 3; ++i) offp[i + 1] = offp[i] + (o->m[i] + pad - 1) / pad * pad;
    if (offp[3] <= 64) break;
    pad = 16;
  }
  const int r = offp[3];
  if (r > PODP_R_MAX)
    return fail(PODP_ERR_UNSUPPORTED, "padded per-direction concatenation (%d) exceeds %d", r, PODP_R_MAX);
  if (!o->N0 || !o->S) return fail(PODP_ERR_ARG, "null N0 / S");
  for (int q = 0; q < 9; ++q)
    if (!o->K[q] || !o->C[q] || !o->H[q] || !o->G[q]) return fail(PODP_ERR_ARG, "null block pointer (index %d)", q);
  for (int i = 0; i < 3; ++i)
    if (!o->b0[i] || !o->b1[i]) return fail(PODP_ERR_ARG, "null b0/b1 pointer (direction %d)", i + 1);
  // (1) the concatenated cross-block operators for the contraction kernel (placement only): K, M block-diagonal
  //     (unused by the solve, which runs on the direction contexts; K's padding diagonal is 1 for validity),
  //     K_R = [K_ij], M_I = [C_ij], b column i in block i, H row i = [h_i^(j)]_j, G placed from the G_ij
  const int ng = 6 + 2 * r;
  std::vector<double> K((size_t)2 * r * r, 0.0), M(K.size(), 0.0), KR(K.size(), 0.0), MI(K.size(), 0.0);
  std::vector<double> B0((size_t)6 * r, 0.0), B1(B0.size(), 0.0), H(B0.size(), 0.0), G((size_t)2 * ng * ng, 0.0);
  for (int i = 0; i < 3; ++i)
    for (int a = o->m[i]; a < offp[i + 1] - offp[i]; ++a) K[2 * ((size_t)(offp[i] + a) * r + offp[i] + a)] = 1.0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      const double *Kb = o->K[3 * i + j], *Cb = o->C[3 * i + j];
      for (int a = 0; a < o->m[i]; ++a)
        for (int b = 0; b < o->m[j]; ++b)
          for (int cc = 0; cc < 2; ++cc) {
            const size_t e = 2 * ((size_t)(offp[i] + a) * r + offp[j] + b) + cc, src = 2 * ((size_t)a * o->m[j] + b) + cc;
            KR[e] = Kb[src];
            MI[e] = Cb[src];
            if (i == j) {
              K[e] = Kb[src];
              M[e] = Cb[src];
            }
          }
      for (int b = 0; b < o->m[j]; ++b)
        for (int cc = 0; cc < 2; ++cc) H[2 * ((size_t)i * r + offp[j] + b) + cc] = o->H[3 * i + j][2 * b + cc];
      // slot map of direction d in the stacked (6 + 2r) factor: [2d, 2d+1 | 6 + offp_d + a | 6 + r + offp_d + a]
      auto slot = [&](int d, int a) { return a < 2 ? 2 * d + a : (a < 2 + o->m[d] ? 6 + offp[d] + (a - 2) : 6 + r + offp[d] + (a - 2 - o->m[d])); };
      const int ni = 2 + 2 * o->m[i], nj = 2 + 2 * o->m[j];
      for (int a = 0; a < ni; ++a)
        for (int b = 0; b < nj; ++b)
          for (int cc = 0; cc < 2; ++cc)
            G[2 * ((size_t)slot(i, a) * ng + slot(j, b)) + cc] = o->G[3 * i + j][2 * ((size_t)a * nj + b) + cc];
    }
  for (int i = 0; i < 3; ++i)
    for (int a = 0; a < o->m[i]; ++a)
      for (int cc = 0; cc < 2; ++cc) {
        B0[2 * ((size_t)(offp[i] + a) * 3 + i) + cc] = o->b0[i][2 * a + cc];
        B1[2 * ((size_t)(offp[i] + a) * 3 + i) + cc] = o->b1[i][2 * a + cc];
      }
  podp_operators emb = {};
  emb.r = r;
  emb.nu = o->nu;
  emb.alpha = o->alpha;
  emb.alpha_lb = o->alpha_lb;
  emb.K = K.data();
  emb.M = M.data();
  emb.K_R = KR.data();
  emb.M_I = MI.data();
  emb.b0 = B0.data();
  emb.b1 = B1.data();
  emb.N0 = o->N0;
  emb.S = o->S;
  emb.H = H.data();
  emb.G = G.data();
  podp_ctx *main_ctx = nullptr;
  podp_status st = podp_create_batch(1, &emb, device, cuda_stream, &main_ctx);
  if (st != PODP_OK) return st;
  // (2) the three direction systems, each its own single-object context of size M_i (exact padding to
  //     8 ceil(M_i / 8): K_pad = diag(K_ii, I), M_pad = diag(C_ii, 0)), right-hand side in column i; their other
  //     operands are unused (zero)
  for (int i = 0; i < 3; ++i) {
    const int mi = o->m[i], ngs = 6 + 2 * mi;
    std::vector<double> zH((size_t)6 * mi, 0.0), zG((size_t)2 * ngs * ngs, 0.0), zS(9, 0.0), eye3(9, 0.0);
    std::vector<double> db0((size_t)6 * mi, 0.0), db1((size_t)6 * mi, 0.0);
    eye3[0] = eye3[4] = eye3[8] = 1.0;
    for (int a = 0; a < mi; ++a)
      for (int cc = 0; cc < 2; ++cc) {
        db0[2 * ((size_t)a * 3 + i) + cc] = o->b0[i][2 * a + cc];
        db1[2 * ((size_t)a * 3 + i) + cc] = o->b1[i][2 * a + cc];
      }
    podp_operators d = {};
    d.r = mi;
    d.nu = o->nu;
    d.alpha = o->alpha;
    d.alpha_lb = o->alpha_lb;
    d.K = o->K[4 * i];
    d.M = o->C[4 * i];
    d.b0 = db0.data();
    d.b1 = db1.data();
    d.N0 = eye3.data();
    d.S = zS.data();
    d.H = zH.data();
    d.G = zG.data();
    st = podp_create_batch(1, &d, device, cuda_stream, &main_ctx->dir[i]);
    if (st != PODP_OK) {
      podp_destroy(main_ctx);
      return st;
    }
  }
  for (int i = 0; i < 3; ++i) {
    main_ctx->m[i] = o->m[i];
    main_ctx->offp[i] = offp[i];
  }
  main_ctx->r = off[3];  // the caller's concatenated size (PODP_FLAG_OUT_P layout, podp_r)
  *out = main_ctx;
  return PODP_OK;
}

}  // extern "C"
