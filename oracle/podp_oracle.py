"""Plain CPU oracle (TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py).

Every function follows one passage of PAPER.md (cited as P:<line>) in the paper's notation, with the BASELINE
sign/shared-basis conventions of SURVEY.md (readings U1-U18 are listed in DESIGN.md).  Loops are explicit; the
only library primitives are numpy.linalg.solve (LAPACK zgesv, partial pivoting) and small dot products.
"""
from __future__ import annotations

import math

import numpy as np

# Output entry order of the 6 unique entries of a symmetric 3x3 tensor: 11, 22, 33, 12, 13, 23.
ENTRY_ORDER = ((0, 0), (1, 1), (2, 2), (0, 1), (0, 2), (1, 2))


def to6(T: np.ndarray) -> np.ndarray:
    return np.array([T[i, j] for (i, j) in ENTRY_ORDER])


def from6(v) -> np.ndarray:
    T = np.zeros((3, 3))
    for e, (i, j) in enumerate(ENTRY_ORDER):
        T[i, j] = T[j, i] = v[e]
    return T


def solve_reduced(K, M, b0, b1, nu: float, omega: float, sign: int = +1) -> np.ndarray:
    """Reduced Galerkin system A^M[omega] p_i = r_i^M[omega], i = 1..3 (eqn:ReducedA).

    BASELINE form (north_star; readings U1-U3): A(omega) = K + i*omega*nu*M (shared basis, one matrix for the
    three directions) and r_i(omega) = b0_i + omega*b1_i (source affine in omega, reading U2).
    Returns P (r x 3), column i = p_i.  LAPACK zgesv (partial pivoting).
    sign=-1 gives the paper's native convention A = K - i omega C, used only by pin C9."""
    s = omega * nu
    A = K + sign * 1j * s * M
    B = b0 + omega * b1
    return np.linalg.solve(A, B)


def mpt_R(P, K_R, alpha: float) -> np.ndarray:
    """(R^PODP)_ij = -(alpha^3/4) conj(p_i)^T K_ij^M p_j (eqn:podprealmpt).

    Real part taken and i <= j mirrored (reading U7: R is real symmetric)."""
    R = np.zeros((3, 3))
    for i in range(3):
        for j in range(i, 3):
            R[i, j] = -(alpha ** 3 / 4.0) * np.real(np.vdot(P[:, i], K_R @ P[:, j]))
            R[j, i] = R[i, j]
    return R


def mpt_I(P, M, S, H, nu: float, alpha: float, omega: float) -> np.ndarray:
    """(I^PODP)_ij of eqn:podpimagmpt, shared-basis form:

    I_ij = (omega alpha^3/4) ( S_ij + Re( conj(p_i)^T C^M p_j + h_i p_j + h_j p_i ) ),  C^M = U^H C U = nu M,
    where S_ij is the precomputed scalar block o_i^T C1 o_j + c_ij + s_i^T o_j + s_j^T o_i
    and h_i the precomputed row o_i^T C2 U + t_i^T U; the conjugated terms of P:614-615 become
    Re(h_j p_i) because Re(conj z) = Re z."""
    I = np.zeros((3, 3))
    pref = omega * alpha ** 3 / 4.0
    for i in range(3):
        for j in range(i, 3):
            quad = np.vdot(P[:, i], (nu * M) @ P[:, j])
            lin = np.dot(H[i], P[:, j]) + np.dot(H[j], P[:, i])
            I[i, j] = pref * (S[i, j] + np.real(quad + lin))
            I[j, i] = I[i, j]
    return I


def residual_coeffs(P, nu: float, omega: float, sign: int = +1) -> np.ndarray:
    """Coefficient vectors w^(i)[omega] of the residual r_i = b0_i + omega b1_i - K U p_i - i omega nu M U p_i in the
    stacked factor [b0_1, b1_1, b0_2, b1_2, b0_3, b1_3 | K U | M U] (SPEC S:488 rewritten for the
    BASELINE Gram).  Returns Wt ((6+2r) x 3)."""
    r = P.shape[0]
    s = omega * nu
    Wt = np.zeros((6 + 2 * r, 3), dtype=np.complex128)
    for i in range(3):
        Wt[2 * i, i] = 1.0
        Wt[2 * i + 1, i] = omega
        Wt[6:6 + r, i] = -P[:, i]
        Wt[6 + r:, i] = -sign * 1j * s * P[:, i]
    return Wt


def certificate(P, G, nu: float, omega: float, alpha: float, alpha_lb: float, sign: int = +1):
    """Lemma 4.1 with the fast residual norms of P:651-661:

    ||r_i||^2 = w_i^H G w_i,  ||r_i - r_j||^2 = ||r_i||^2 + ||r_j||^2 - 2 Re(w_i^H G w_j),
    Delta_ij = alpha^3/(8 alpha_LB) (||r_i||^2 + ||r_j||^2 + ||r_i - r_j||^2).
    Squared norms clamped at 0 (reading U10).  Returns (Delta 3x3, n (3,), X 3x3)."""
    Wt = residual_coeffs(P, nu, omega, sign)
    X = np.zeros((3, 3), dtype=np.complex128)
    for i in range(3):
        for j in range(3):
            X[i, j] = np.vdot(Wt[:, i], G @ Wt[:, j])
    n = np.array([max(0.0, float(np.real(X[i, i]))) for i in range(3)])
    D = np.zeros((3, 3))
    for i in range(3):
        for j in range(i, 3):
            m = max(0.0, n[i] + n[j] - 2.0 * float(np.real(X[i, j]))) if i != j else 0.0
            D[i, j] = alpha ** 3 / (8.0 * alpha_lb) * (n[i] + n[j] + m)
            D[j, i] = D[i, j]
    return D, n, X


def evaluate_one(ops, omega: float, out_R: bool = False, sign: int = +1) -> dict:
    """Algorithm 1 on-line body for one output frequency (alg:adapt lines 23-26) plus the certificate.

    Returns dict(P, T1 (Rt = N0 + R, or R if out_R), R, I, Delta) with 3x3 tensors."""
    K_R = ops.K if ops.K_R is None else ops.K_R
    P = solve_reduced(ops.K, ops.M, ops.b0, ops.b1, ops.nu, omega, sign)
    R = mpt_R(P, K_R, ops.alpha)
    I = mpt_I(P, ops.M, ops.S, ops.H, ops.nu, ops.alpha, omega)
    D, _, _ = certificate(P, ops.G, ops.nu, omega, ops.alpha, ops.alpha_lb, sign)
    T1 = R if out_R else np.asarray(ops.N0, dtype=float) + R
    return dict(P=P, T1=T1, R=R, I=I, Delta=D)


def evaluate(ops, omegas, out_R: bool = False):
    """Sweep over output frequencies (Algorithm 1 lines 22-26).  Returns (T1, I, Delta), each F x 6 in ENTRY_ORDER."""
    F = len(omegas)
    T1 = np.zeros((F, 6))
    I = np.zeros((F, 6))
    D = np.zeros((F, 6))
    for f, w in enumerate(omegas):
        out = evaluate_one(ops, float(w), out_R=out_R)
        T1[f], I[f], D[f] = to6(out["T1"]), to6(out["I"]), to6(out["Delta"])
    return T1, I, D


def select(omegas, Delta6, snap, n_star: int, theta: float | None = None):
    """One greedy step of Algorithm 1 ("at most one additional snapshot per interval").

    Intervals [snap_n, snap_{n+1}), the last one closed (reading U12); grid points equal to a snapshot are not
    candidates; empty intervals are skipped.  Lambda_n = max over in-interval omega and over i<=j of Delta_ij
    (NaN entries ignored); the N* intervals with largest Lambda_n are chosen (ties: lower interval index), and
    within an interval the argmax is the lowest grid index (reading U13).
    theta in (0, 1] selects the variant of P:698 instead: every interval with Lambda_n >= theta * Lambda (at most
    n_star of them, largest first).
    Returns (omega_new ascending, idx_new, Lambda_global, Lambda_n list (None for empty))."""
    snap = [float(x) for x in snap]
    n_int = len(snap) - 1
    lam = [None] * n_int
    arg = [None] * n_int
    snapset = set(snap)
    for f in range(len(omegas)):
        w = float(omegas[f])
        if w in snapset:
            continue
        n = None
        for t in range(n_int):
            last = (t == n_int - 1)
            if snap[t] <= w and (w < snap[t + 1] or (last and w <= snap[t + 1])):
                n = t
                break
        if n is None:
            continue
        for e in range(6):
            d = float(Delta6[f][e])
            if d != d:  # NaN
                continue
            if lam[n] is None or d > lam[n]:
                lam[n] = d
                arg[n] = f
    cands = [t for t in range(n_int) if lam[t] is not None]
    if theta is None and len(cands) < n_star:
        raise ValueError("fewer non-empty intervals than n_star")
    if not cands:
        raise ValueError("no candidates")
    Lam = max(lam[t] for t in cands)
    if theta is not None:
        cands = [t for t in cands if lam[t] >= theta * Lam]
    order = sorted(cands, key=lambda t: (-lam[t], t))[:n_star]
    idx = sorted(arg[t] for t in order)
    return [float(omegas[f]) for f in idx], idx, Lam, lam


def invariants(T6) -> tuple:
    """Rotation invariants of the MPT: ascending eigenvalues of Rt and of I (numpy.linalg.eigvalsh on the
    3x3 symmetric blocks).  T6: (n, 6) pair (Rt6, I6).  Returns (n x 3, n x 3)."""
    R6, I6 = T6
    eR = np.array([np.linalg.eigvalsh(from6(r)) for r in R6])
    eI = np.array([np.linalg.eigvalsh(from6(i)) for i in I6])
    return eR, eI


def coil_voltage(Rt6, I6, h_ex, h_ms):
    """eqn:meas_voltage: V = (H0^ms)_i M_ij (H0)_j with M = Rt + i I.  Returns (n, n_coil) complex."""
    out = np.zeros((len(Rt6), len(h_ex)), dtype=np.complex128)
    for f in range(len(Rt6)):
        Mx = from6(Rt6[f]) + 1j * from6(I6[f])
        for c in range(len(h_ex)):
            out[f, c] = np.asarray(h_ms[c]) @ Mx @ np.asarray(h_ex[c])
    return out
