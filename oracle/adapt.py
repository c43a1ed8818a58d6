"""Algorithm 1 (alg:adapt) on a synthetic full-order system -- TEST INFRASTRUCTURE ONLY (see
oracle/__init__.py).  Plain NumPy, step by step in the paper's order; the on-line body is oracle.evaluate and the
greedy step is oracle.select.

Readings (N2): shared basis (one TSVD of D = [D_1 D_2 D_3], reading U3); TSVD keeps the
s_k with s_k / s_1 >= TOL_Sigma (P:584 is garbled: "largest singular value such that s_M/s_1 < TOL"); the first
certification happens before the loop test (line 8 needs a Lambda); |B_alpha| is an input (default 1).
"""
from __future__ import annotations

import numpy as np

from .perdir import PerDirectionROM, tsvd_per_direction
from .podp_oracle import evaluate, select


def full_solve(fom, omega: float) -> np.ndarray:
    """Line 4 / line 16: q_i[omega] from eqn:Linear, dense LAPACK.  N x 3."""
    A = fom.K_full + 1j * omega * fom.nu * fom.M_full
    return np.linalg.solve(A, fom.B0f + omega * fom.B1f)


def tsvd(D: np.ndarray, tol_sigma: float) -> np.ndarray:
    """Lines 6 / 19: D^M = U^M Sigma^M (V^M)^H, keeping s_1..s_M with s_M / s_1 >= TOL_Sigma."""
    U, s, _ = np.linalg.svd(D, full_matrices=False)
    M = int(np.sum(s / s[0] >= tol_sigma))
    return U[:, :M]


def reduced_operators(fom, U: np.ndarray):
    """Projected operators: K = U^H K U, M = U^H M U (M is the nu-free C), b = U^H B, N0 = I (synthetic
    mu_r = 1 reading), S = v^T C v, H = v^T C U, and the residual Gram G = W^H W with
    W = [B0f_1, B1f_1, B0f_2, B1f_2, B0f_3, B1f_3 | K U | M U] (Lemma 4.1's fast form)."""
    from podp_inputs.generators import Operators
    N, r = U.shape
    Uh = U.conj().T
    K = Uh @ fom.K_full @ U
    M = Uh @ fom.M_full @ U
    W = np.zeros((N, 6 + 2 * r), dtype=np.complex128)
    for i in range(3):
        W[:, 2 * i] = fom.B0f[:, i]
        W[:, 2 * i + 1] = fom.B1f[:, i]
    W[:, 6:6 + r] = fom.K_full @ U
    W[:, 6 + r:] = fom.M_full @ U
    G = W.conj().T @ W
    S = np.real(fom.v.T @ fom.C_full @ fom.v)
    return Operators(K=0.5 * (K + K.conj().T), M=0.5 * (M + M.conj().T), b0=Uh @ fom.B0f, b1=Uh @ fom.B1f,
                     N0=np.eye(3), S=0.5 * (S + S.T), H=fom.v.T @ fom.C_full @ U, G=0.5 * (G + G.conj().T),
                     nu=fom.nu, alpha=fom.alpha, alpha_lb=fom.alpha_lb)


def run_adaptive(fom, omegas, n0: int = 13, n_star: int = 2, tol_sigma: float = 1e-6, tol_delta: float = 1e-3,
                 max_k: int = 4, vol: float = 1.0, theta: float | None = None, snap0=None,
                 per_direction: bool = False):
    """Algorithm 1 lines 1-26.  Returns (ops, (T1, I, Delta) on omegas, history) where history[k-1] =
    dict(k, N, r, Lambda, snap (sorted), new (omegas chosen at this k, empty at the last))."""
    from podp_inputs.generators import snapshot_grid
    snap = [float(w) for w in (snapshot_grid(n0) if snap0 is None else snap0)]          # line 3
    Q = {w: full_solve(fom, w) for w in snap}                                             # line 4
    k = 1
    history = []
    while True:
        if per_direction:                                                                # N1: D_i, U_i^M
            Us = tsvd_per_direction([Q[w] for w in snap], tol_sigma)
            ops = PerDirectionROM(fom, Us)
            T1, I, Dl = ops.evaluate(omegas)
            m = [U.shape[1] for U in Us]
        else:
            D = np.concatenate([Q[w] for w in snap], axis=1)                             # lines 5 / 18
            U = tsvd(D, tol_sigma)                                                       # lines 6 / 19
            ops = reduced_operators(fom, U)
            T1, I, Dl = evaluate(ops, omegas)                                            # line 11
            m = [U.shape[1]]
        new, _idx, Lam, _lam = select(omegas, Dl, snap, n_star, theta)                   # lines 12-15
        rec = dict(k=k, N=len(snap), r=sum(m), m=m, Lambda=Lam, snap=list(snap), new=[])
        history.append(rec)
        if not (Lam / vol > tol_delta and k < max_k):                                    # line 8
            return ops, (T1, I, Dl), history
        k += 1                                                                           # line 9
        rec["new"] = list(new)
        for w in new:                                                                    # line 16
            Q[w] = full_solve(fom, w)
        snap = sorted(snap + list(new))                                                  # line 17
