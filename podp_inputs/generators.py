"""Seeded generators (see package docstring).  All complex data complex128, row-major (C order).

Draw order is part of the contract; changing it changes every seeded input.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

MU0 = 4.0 * math.pi * 1e-7  # PAPER.md P:159, mu_0 = 4 pi 1e-7 exactly (reading U15)
# BASELINE.json configs[0]: nu = mu0 * sigma * alpha^2 = 4 pi 1e-7 * 5.96e7 * (1e-2)^2 (omega-free; paper's nu-tilde)
NU_DEFAULT = MU0 * 5.96e7 * (1e-2) ** 2
ALPHA_DEFAULT = 1e-2


@dataclasses.dataclass
class Operators:
    """Inputs of podp_create for one object (shared reduced basis, BASELINE form).

    K, M, K_R: r x r Hermitian; b0, b1: r x 3 (column i = direction i); N0, S: 3 x 3 real symmetric;
    H: 3 x r (row i = h_i, unconjugated); G: (6+2r) x (6+2r) Hermitian PSD Gram, slot order
    [b0_1, b1_1, b0_2, b1_2, b0_3, b1_3 | K U (r) | M U (r)].
    """
    K: np.ndarray
    M: np.ndarray
    b0: np.ndarray
    b1: np.ndarray
    N0: np.ndarray
    S: np.ndarray
    H: np.ndarray
    G: np.ndarray
    nu: float
    alpha: float
    alpha_lb: float
    K_R: np.ndarray | None = None

    @property
    def r(self) -> int:
        return int(self.K.shape[0])

    def copy(self) -> "Operators":
        return dataclasses.replace(self, **{f.name: (np.array(getattr(self, f.name)) if isinstance(getattr(self, f.name), np.ndarray) else getattr(self, f.name))
                                            for f in dataclasses.fields(self)})


@dataclasses.dataclass
class Config0Extras:
    """Full-order objects of the tiny config 0 (oracle-side full-order checks only)."""
    K_full: np.ndarray
    M_full: np.ndarray
    C_full: np.ndarray       # nu * M_full
    U: np.ndarray            # N x r orthonormal
    v: np.ndarray            # N x 3 real (theta0-tilde + e_i x xi coefficients, conductor dofs)
    B0f: np.ndarray          # N x 3 full-order source, omega^0 part
    B1f: np.ndarray          # N x 3 full-order source, omega^1 part
    W: np.ndarray            # N x (6+2r) residual factor, G = W^H W


def cn(rng: np.random.Generator, shape, var: float) -> np.ndarray:
    """CN(0, var): sqrt(var/2) * (N(0,1) + i N(0,1)); the whole real array is drawn first (reading U16)."""
    re = rng.standard_normal(shape)
    im = rng.standard_normal(shape)
    return math.sqrt(var / 2.0) * (re + 1j * im)


def _herm(X: np.ndarray) -> np.ndarray:
    return 0.5 * (X + X.conj().T)


def omega_grid(F: int, lo: float = 1e1, hi: float = 1e8) -> np.ndarray:
    """F log-spaced output frequencies on [lo, hi] rad/s (BASELINE configs)."""
    return np.logspace(math.log10(lo), math.log10(hi), F)


def snapshot_grid(N: int = 13, lo: float = 1e1, hi: float = 1e8) -> np.ndarray:
    """Initial log-spaced snapshot set, N = 13 on [1e1, 1e8] (Algorithm 1 line 3; reading U14)."""
    return np.logspace(math.log10(lo), math.log10(hi), N)


def embed_gram(G1: np.ndarray, r: int) -> np.ndarray:
    """Embed the literal (2+2r) Gram into the stacked (6+2r) slot order (reading U9): G[u,v] = G1[pi(u), pi(v)]."""
    pi = np.array([0, 1, 0, 1, 0, 1] + list(range(2, 2 + 2 * r)))
    return G1[np.ix_(pi, pi)].copy()


def make_operators(r: int, seed: int = 0, nu: float = NU_DEFAULT, alpha: float = ALPHA_DEFAULT,
                   alpha_lb: float = 1.0) -> Operators:
    """Config 1/2/4 generator (BASELINE.json configs[1]; SURVEY.md 8(d) draw order (1)..(6))."""
    if r < 2 or r % 2:
        raise ValueError("r must be even and >= 2 (M has rank r/2)")
    rng = np.random.default_rng(seed)
    B = cn(rng, (r, r), 1.0 / r)
    K = _herm(B @ B.conj().T + r * np.eye(r))
    C = cn(rng, (r, r // 2), 1.0 / r)
    M = _herm(C @ C.conj().T)
    b0 = cn(rng, (r, 3), 1.0)
    b1 = cn(rng, (r, 3), 1.0)
    Sr = rng.standard_normal((3, 3))
    S = np.triu(Sr) + np.triu(Sr, 1).T
    H = cn(rng, (3, r), 1.0)
    W = cn(rng, (2 * (2 + 2 * r), 2 + 2 * r), 1.0)
    G1 = W.conj().T @ W
    G = embed_gram(G1, r)
    return Operators(K=K, M=M, b0=b0, b1=b1, N0=np.eye(3), S=S, H=H, G=G, nu=float(nu), alpha=float(alpha),
                     alpha_lb=float(alpha_lb))


def make_pivot_forcing(r: int, seed: int = 0) -> Operators:
    """Test input that REQUIRES row interchanges: K = [[0, B], [B^H, 0]] Hermitian indefinite
    with an exactly zero leading block, M = diag(0, C C^H) PSD, so A(omega) = K + i omega nu M has a zero (r/2 x r/2)
    leading block at every omega: LU without pivoting meets an exactly zero pivot at step 0, partial pivoting does
    not.  Everything else as make_operators(r, seed)."""
    if r < 2 or r % 2:
        raise ValueError("r must be even and >= 2")
    base = make_operators(r, seed)
    rng = np.random.default_rng(10_000 + seed)
    h = r // 2
    B = cn(rng, (h, h), 1.0) + 2.0 * np.eye(h)
    K = np.zeros((r, r), complex)
    K[:h, h:] = B
    K[h:, :h] = B.conj().T
    C = cn(rng, (h, max(1, h // 2)), 1.0 / h)
    M = np.zeros((r, r), complex)
    M[h:, h:] = _herm(C @ C.conj().T)
    return Operators(**{**base.__dict__, "K": _herm(K), "M": M})


def make_illconditioned(r: int, kappa: float = 1e8, seed: int = 0) -> Operators:
    """Hermitian positive definite K with condition number kappa (spectrum log-spaced on [1, kappa] in a random
    unitary basis); everything else as make_operators(r, seed).  For the pencil path (N3), whose Z = L^{-H} V has
    condition number sqrt(kappa(K))."""
    base = make_operators(r, seed)
    rng = np.random.default_rng(20_000 + seed)
    Q, _ = np.linalg.qr(cn(rng, (r, r), 1.0))
    lam = np.logspace(0.0, math.log10(kappa), r)
    K = _herm((Q * lam) @ Q.conj().T)
    return Operators(**{**base.__dict__, "K": K})


def make_perdir_blocks(m=(16, 16, 16), seed: int = 0, nu: float = NU_DEFAULT, alpha: float = ALPHA_DEFAULT,
                       alpha_lb: float = 1.0) -> dict:
    """Per-direction operator blocks for the literal N1 path (timing / GPU tests), drawn like make_operators on
    the concatenated space n = M_1 + M_2 + M_3 and cut into blocks: K = B B^H + n I, M = C C^H (rank n/2),
    Kb[i][j] / Cb[i][j] its M_i x M_j blocks; b0[i], b1[i] ~ CN(0,1); Hb[i][j] ~ CN(0,1) rows; S symmetric N(0,1);
    Gx[i][j] the blocks of W^H W (W ~ CN(0,1)) on direction i's slots [b0_i, b1_i | KU_i | MU_i] (a consistent
    PSD Gram).  Draws only -- no on-line arithmetic."""
    rng = np.random.default_rng(seed)
    m = [int(x) for x in m]
    n = sum(m)
    off = np.concatenate([[0], np.cumsum(m)])
    B = cn(rng, (n, n), 1.0 / n)
    K = _herm(B @ B.conj().T + n * np.eye(n))
    C = cn(rng, (n, max(1, n // 2)), 1.0 / n)
    M = _herm(C @ C.conj().T)
    b0 = [cn(rng, (m[i],), 1.0) for i in range(3)]
    b1 = [cn(rng, (m[i],), 1.0) for i in range(3)]
    Hb = [[cn(rng, (m[j],), 1.0) for j in range(3)] for _i in range(3)]
    S = rng.standard_normal((3, 3))
    S = np.triu(S) + np.triu(S, 1).T
    W = cn(rng, (2 * (6 + 2 * n), 6 + 2 * n), 1.0)
    Gf = _herm(W.conj().T @ W)
    slots = [np.concatenate([[2 * i, 2 * i + 1], 6 + np.arange(off[i], off[i + 1]),
                             6 + n + np.arange(off[i], off[i + 1])]) for i in range(3)]
    blk = lambda X, i, j: X[off[i]:off[i + 1], off[j]:off[j + 1]]  # noqa: E731
    return dict(m=m, Kb=[[blk(K, i, j) for j in range(3)] for i in range(3)],
                Cb=[[blk(M, i, j) for j in range(3)] for i in range(3)], b0=b0, b1=b1, Hb=Hb, N0=np.eye(3), S=S,
                Gx=[[Gf[np.ix_(slots[i], slots[j])] for j in range(3)] for i in range(3)], nu=nu, alpha=alpha,
                alpha_lb=alpha_lb)


def batch_sigma(n_obj: int = 256) -> np.ndarray:
    """Config 3 conductivities: log-uniform in [1e6, 6e7] S/m from a separate stream (SURVEY 8(d) proposal)."""
    return 10.0 ** np.random.default_rng(0).uniform(6.0, math.log10(6e7), n_obj)


def make_config0(seed: int = 0, N: int = 2000, r: int = 8, nu: float = NU_DEFAULT, alpha: float = ALPHA_DEFAULT,
                 alpha_lb: float = 0.1):
    """Tiny config 0: synthetic full-order system N=2000 projected onto an orthonormal U (BASELINE configs[0]).

    Returns (Operators, Config0Extras). Draw order (1)..(8) of SURVEY.md 8(d).
    """
    rng = np.random.default_rng(seed)
    nnz_per_row = 8
    cols = rng.integers(0, N, nnz_per_row * N)
    vals = cn(rng, (nnz_per_row * N,), 1.0)
    A = np.zeros((N, N), dtype=np.complex128)
    rows = np.repeat(np.arange(N), nnz_per_row)
    np.add.at(A, (rows, cols), vals)
    K_full = _herm(A.conj().T @ A + 0.1 * np.eye(N))
    Nc = N // 2
    Cc = cn(rng, (1000, Nc), 1.0)
    M_full = np.zeros((N, N), dtype=np.complex128)
    M_full[:Nc, :Nc] = Cc.conj().T @ Cc
    M_full = _herm(M_full)
    U, _ = np.linalg.qr(cn(rng, (N, r), 1.0))
    K = _herm(U.conj().T @ K_full @ U)
    M = _herm(U.conj().T @ M_full @ U)
    b0 = cn(rng, (r, 3), 1.0)
    b1 = cn(rng, (r, 3), 1.0)
    v = np.zeros((N, 3))
    v[:Nc] = rng.standard_normal((Nc, 3))
    C_full = nu * M_full
    S = np.real(v.T @ C_full @ v)
    S = 0.5 * (S + S.T)
    H = v.T @ C_full @ U
    z0 = cn(rng, (N, 3), 1.0)
    z1 = cn(rng, (N, 3), 1.0)
    Pperp = lambda z: z - U @ (U.conj().T @ z)  # noqa: E731
    B0f = U @ b0 + Pperp(z0)
    B1f = U @ b1 + Pperp(z1)
    W = np.zeros((N, 6 + 2 * r), dtype=np.complex128)
    for i in range(3):
        W[:, 2 * i] = B0f[:, i]
        W[:, 2 * i + 1] = B1f[:, i]
    W[:, 6:6 + r] = K_full @ U
    W[:, 6 + r:] = M_full @ U
    G = _herm(W.conj().T @ W)
    ops = Operators(K=K, M=M, b0=b0, b1=b1, N0=np.eye(3), S=S, H=H, G=G, nu=float(nu), alpha=float(alpha),
                    alpha_lb=float(alpha_lb))
    return ops, Config0Extras(K_full=K_full, M_full=M_full, C_full=C_full, U=U, v=v, B0f=B0f, B1f=B1f, W=W)


def make_galerkin_variant(ops: Operators, ex: Config0Extras, seed: int = 1):
    """Pin C3 input: b0 = U^H K_full U y, b1 = i nu U^H M_full U y with full-order sources in span(K U y), so the
    exact full-order solution is U y for every omega.  Returns (ops', ex', y)."""
    rng = np.random.default_rng(seed)
    r = ops.r
    y = cn(rng, (r, 3), 1.0)
    B0f = ex.K_full @ (ex.U @ y)
    B1f = 1j * ops.nu * (ex.M_full @ (ex.U @ y))
    b0 = ex.U.conj().T @ B0f
    b1 = ex.U.conj().T @ B1f
    W = ex.W.copy()
    for i in range(3):
        W[:, 2 * i] = B0f[:, i]
        W[:, 2 * i + 1] = B1f[:, i]
    G = _herm(W.conj().T @ W)
    ops2 = dataclasses.replace(ops, b0=b0, b1=b1, G=G)
    ex2 = dataclasses.replace(ex, B0f=B0f, B1f=B1f, W=W)
    return ops2, ex2, y


def make_identity_basis_variant(seed: int = 0, r: int = 8, nu: float = NU_DEFAULT, alpha: float = ALPHA_DEFAULT):
    """Pin C5 input: N = r, U = I (full order == reduced order)."""
    return make_config0(seed=seed, N=2 * r, r=r, nu=nu, alpha=alpha)  # N=2r keeps a conductor half; U from QR


def pad_operators(ops: Operators, r_pad: int) -> Operators:
    """Exact padding: K_pad = diag(K, I); M, K_R, b, H, G zero-padded (G in both r-blocks)."""
    r = ops.r
    if r_pad < r:
        raise ValueError("r_pad < r")
    def pad_sq(X, eye):
        Y = np.zeros((r_pad, r_pad), dtype=np.complex128)
        Y[:r, :r] = X
        if eye:
            Y[r:, r:] = np.eye(r_pad - r)
        return Y
    def pad_rows(X):
        Y = np.zeros((r_pad, X.shape[1]), dtype=np.complex128)
        Y[:r] = X
        return Y
    H = np.zeros((3, r_pad), dtype=np.complex128)
    H[:, :r] = ops.H
    n, n2 = 6 + 2 * r, 6 + 2 * r_pad
    idx = np.concatenate([np.arange(6), 6 + np.arange(r), 6 + r_pad + np.arange(r)])
    G = np.zeros((n2, n2), dtype=np.complex128)
    G[np.ix_(idx, idx)] = ops.G[:n, :n]
    return dataclasses.replace(ops, K=pad_sq(ops.K, True), M=pad_sq(ops.M, False),
                               K_R=None if ops.K_R is None else pad_sq(ops.K_R, False),
                               b0=pad_rows(ops.b0), b1=pad_rows(ops.b1), H=H, G=G)


_CONFIGS = {
    0: dict(name="c0_tiny_r8_F200", r=8, F=200, n_obj=1),
    1: dict(name="c1_r24_F1e4", r=24, F=10_000, n_obj=1),
    2: dict(name="c2_r48_F1e5", r=48, F=100_000, n_obj=1),
    3: dict(name="c3_dict256_r32_F2000", r=32, F=2_000, n_obj=256),
    4: dict(name="c4_r96_F1e6_select", r=96, F=1_000_000, n_obj=1, n_snap=13, n_star=2),
}


def config_spec(k: int) -> dict:
    return dict(_CONFIGS[k])


def make_config(k: int, F: int | None = None, n_obj: int | None = None):
    """Return dict(spec, ops=[Operators per object], omega, extras) for BASELINE config k (F/n_obj overridable)."""
    spec = config_spec(k)
    if F is not None:
        spec["F"] = int(F)
    if n_obj is not None:
        spec["n_obj"] = int(n_obj)
    omega = omega_grid(spec["F"])
    extras = None
    if k == 0:
        ops, extras = make_config0()
        ops_list = [ops]
    elif k == 3:
        sig = batch_sigma(256)
        ops_list = [make_operators(spec["r"], seed=j, nu=MU0 * sig[j] * ALPHA_DEFAULT ** 2) for j in range(spec["n_obj"])]
    else:
        ops_list = [make_operators(spec["r"], seed=0)]
    out = dict(spec=spec, ops=ops_list, omega=omega, extras=extras)
    if k == 4:
        out["snap"] = snapshot_grid(spec["n_snap"])
    return out


@dataclasses.dataclass
class FullOrderSystem:
    """Synthetic full-order system for the Algorithm-1 driver (NEXT row N2).

    (K_full + i omega nu M_full) q_i = B0f_i + omega B1f_i  (eqn:Linear P:476-483, BASELINE sign), C_full = nu M_full,
    v: N x 3 real conductor coefficients (theta0-tilde + e_i x xi), so S = v^T C v and H = v^T C U."""
    K_full: np.ndarray
    M_full: np.ndarray
    C_full: np.ndarray
    v: np.ndarray
    B0f: np.ndarray
    B1f: np.ndarray
    nu: float
    alpha: float
    alpha_lb: float

    @property
    def N(self) -> int:
        return int(self.K_full.shape[0])


def make_fullorder(seed: int = 0, N: int = 1000, n_modes: int = 120, w_lo: float = 1e2, w_hi: float = 1e7,
                   b0_scale: float = 0.1, nu: float = NU_DEFAULT, alpha: float = ALPHA_DEFAULT,
                   alpha_lb: float = 0.1) -> FullOrderSystem:
    """Full-order recipe with the spectral structure of an MPT signature (sum of first-order relaxation terms,
    Lemma 8.5 / P:928): K_full = A^H A + 0.1 I (A sparse, 8 CN(0,1) entries per row), M_full = X diag(lam) X^H of
    rank n_modes supported on the conductor half, lam log-spaced so the relaxation frequencies 1/(nu lam) fall in
    [w_lo, w_hi]; B1f = -i nu M_full v (the source is omega times the conductor term, so q -> -v as omega -> inf,
    P:437 with the omega-free nu); B0f = b0_scale CN(0,1) (the omega-independent mu_r-contrast term).
    Draw order: (1) A columns, (2) A values, (3) X, (4) v, (5) B0f."""
    rng = np.random.default_rng(seed)
    nnz_per_row = 8
    cols = rng.integers(0, N, nnz_per_row * N)
    vals = cn(rng, (nnz_per_row * N,), 1.0)
    A = np.zeros((N, N), dtype=np.complex128)
    np.add.at(A, (np.repeat(np.arange(N), nnz_per_row), cols), vals)
    K_full = _herm(A.conj().T @ A + 0.1 * np.eye(N))
    Nc = N // 2
    X = np.zeros((N, n_modes), dtype=np.complex128)
    X[:Nc] = cn(rng, (Nc, n_modes), 1.0 / Nc)
    lam = np.logspace(math.log10(1.0 / (nu * w_lo)), math.log10(1.0 / (nu * w_hi)), n_modes)
    M_full = _herm((X * lam) @ X.conj().T)
    v = np.zeros((N, 3))
    v[:Nc] = rng.standard_normal((Nc, 3))
    B0f = b0_scale * cn(rng, (N, 3), 1.0)
    B1f = -1j * nu * (M_full @ v)
    return FullOrderSystem(K_full=K_full, M_full=M_full, C_full=nu * M_full, v=v, B0f=B0f, B1f=B1f, nu=float(nu),
                           alpha=float(alpha), alpha_lb=float(alpha_lb))
