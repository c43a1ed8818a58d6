// Host-side, omega-independent precompute for the pencil solver (NEXT row N3 of SURVEY 8(f)), part of row a1.
//
// For K Hermitian positive definite:  K = L L^H (Cholesky),  L^{-1} M L^{-H} = V diag(lambda) V^H (Hermitian
// eigendecomposition, cyclic complex Jacobi),  Z = L^{-H} V.  Then Z^H K Z = I, Z^H M Z = diag(lambda) and
//     A(omega)^{-1} = Z (I + i omega nu diag(lambda))^{-1} Z^H,
// so P(omega) = Z diag(1/(1 + i s lambda_k)) (c0 + omega c1) with c0 = Z^H b0, c1 = Z^H b1, s = omega nu --
// an exact reformulation of the reduced solve of eqn:ReducedA costing O(r^2) per frequency instead of
// the LU's O(r^3) ("the cost of solving ... is at most O(M^3)").
#include <cmath>
#include <complex>
#include <vector>

#include "podp_internal.h"

namespace podp {

using cd = std::complex<double>;

static inline cd C(const double *X, int ld, int i, int j) { return cd(X[2 * ((size_t)i * ld + j)], X[2 * ((size_t)i * ld + j) + 1]); }

// Cyclic Jacobi for a Hermitian n x n matrix (row-major, modified in place): eigenvalues lam, eigenvectors V
// (columns).  Each rotation zeroes A[p][q] with the unitary G = [[c, -s e^{i phi}], [s e^{-i phi}, c]].
static void jacobi_herm(int n, std::vector<cd> &A, std::vector<double> &lam, std::vector<cd> &V) {
  V.assign((size_t)n * n, cd(0.0, 0.0));
  for (int i = 0; i < n; ++i) V[(size_t)i * n + i] = 1.0;
  auto a = [&](int i, int j) -> cd & { return A[(size_t)i * n + j]; };
  double fro = 0.0;
  for (auto &x : A) fro += std::norm(x);
  fro = std::sqrt(fro);
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < n; ++p)
      for (int q = 0; q < n; ++q)
        if (p != q) off += std::norm(a(p, q));
    if (std::sqrt(off) <= 1e-15 * fro || off == 0.0) break;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        const cd apq = a(p, q);
        const double mag = std::abs(apq);
        if (mag == 0.0) continue;
        const cd ph = apq / mag;
        const double theta = 0.5 * std::atan2(2.0 * mag, a(p, p).real() - a(q, q).real());
        const double c = std::cos(theta), s = std::sin(theta);
        for (int i = 0; i < n; ++i) {  // columns: A <- A G
          const cd xp = a(i, p), xq = a(i, q);
          a(i, p) = c * xp + s * std::conj(ph) * xq;
          a(i, q) = -s * ph * xp + c * xq;
        }
        for (int j = 0; j < n; ++j) {  // rows: A <- G^H A
          const cd xp = a(p, j), xq = a(q, j);
          a(p, j) = c * xp + s * ph * xq;
          a(q, j) = -s * std::conj(ph) * xp + c * xq;
        }
        for (int i = 0; i < n; ++i) {
          const cd vp = V[(size_t)i * n + p], vq = V[(size_t)i * n + q];
          V[(size_t)i * n + p] = c * vp + s * std::conj(ph) * vq;
          V[(size_t)i * n + q] = -s * ph * vp + c * vq;
        }
      }
  }
  lam.resize(n);
  for (int i = 0; i < n; ++i) lam[i] = a(i, i).real();
}

bool pencil_precompute(int r, const double *K, const double *M, const double *b0, const double *b1,
                       std::vector<double> &Zo, std::vector<double> &lamo, std::vector<double> &c0o,
                       std::vector<double> &c1o) {
  const int n = r;
  // Cholesky K = L L^H (lower L)
  std::vector<cd> L((size_t)n * n, cd(0.0, 0.0));
  for (int j = 0; j < n; ++j) {
    double d = C(K, n, j, j).real();
    for (int k = 0; k < j; ++k) d -= std::norm(L[(size_t)j * n + k]);
    if (!(d > 0.0)) return false;
    const double ljj = std::sqrt(d);
    L[(size_t)j * n + j] = ljj;
    for (int i = j + 1; i < n; ++i) {
      cd v = C(K, n, i, j);
      for (int k = 0; k < j; ++k) v -= L[(size_t)i * n + k] * std::conj(L[(size_t)j * n + k]);
      L[(size_t)i * n + j] = v / ljj;
    }
  }
  // X = L^{-1} M (forward substitution, column by column)
  std::vector<cd> X((size_t)n * n);
  for (int col = 0; col < n; ++col)
    for (int i = 0; i < n; ++i) {
      cd v = C(M, n, i, col);
      for (int k = 0; k < i; ++k) v -= L[(size_t)i * n + k] * X[(size_t)k * n + col];
      X[(size_t)i * n + col] = v / L[(size_t)i * n + i];
    }
  // Mt = X L^{-H} = (L^{-1} X^H)^H : Y = L^{-1} X^H, Mt = Y^H
  std::vector<cd> Y((size_t)n * n), Mt((size_t)n * n);
  for (int col = 0; col < n; ++col)
    for (int i = 0; i < n; ++i) {
      cd v = std::conj(X[(size_t)col * n + i]);  // (X^H)[i][col]
      for (int k = 0; k < i; ++k) v -= L[(size_t)i * n + k] * Y[(size_t)k * n + col];
      Y[(size_t)i * n + col] = v / L[(size_t)i * n + i];
    }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) Mt[(size_t)i * n + j] = std::conj(Y[(size_t)j * n + i]);
  for (int i = 0; i < n; ++i)  // exact Hermitian symmetrisation before Jacobi
    for (int j = i; j < n; ++j) {
      const cd h = 0.5 * (Mt[(size_t)i * n + j] + std::conj(Mt[(size_t)j * n + i]));
      Mt[(size_t)i * n + j] = h;
      Mt[(size_t)j * n + i] = std::conj(h);
    }
  std::vector<double> lam;
  std::vector<cd> V;
  jacobi_herm(n, Mt, lam, V);
  // Z = L^{-H} V (back substitution with L^H, upper)
  std::vector<cd> Z((size_t)n * n);
  for (int col = 0; col < n; ++col)
    for (int i = n - 1; i >= 0; --i) {
      cd v = V[(size_t)i * n + col];
      for (int k = i + 1; k < n; ++k) v -= std::conj(L[(size_t)k * n + i]) * Z[(size_t)k * n + col];
      Z[(size_t)i * n + col] = v / std::conj(L[(size_t)i * n + i]);
    }
  Zo.resize((size_t)2 * n * n);
  for (size_t e = 0; e < (size_t)n * n; ++e) {
    Zo[2 * e] = Z[e].real();
    Zo[2 * e + 1] = Z[e].imag();
  }
  lamo = lam;
  // c = Z^H b (direction-major 3 x n)
  c0o.assign((size_t)6 * n, 0.0);
  c1o.assign((size_t)6 * n, 0.0);
  for (int c3 = 0; c3 < 3; ++c3)
    for (int k = 0; k < n; ++k) {
      cd s0(0.0, 0.0), s1(0.0, 0.0);
      for (int i = 0; i < n; ++i) {
        const cd zc = std::conj(Z[(size_t)i * n + k]);
        s0 += zc * C(b0, 3, i, c3);
        s1 += zc * C(b1, 3, i, c3);
      }
      c0o[2 * ((size_t)c3 * n + k)] = s0.real();
      c0o[2 * ((size_t)c3 * n + k) + 1] = s0.imag();
      c1o[2 * ((size_t)c3 * n + k)] = s1.real();
      c1o[2 * ((size_t)c3 * n + k) + 1] = s1.imag();
    }
  return true;
}

}  // namespace podp
