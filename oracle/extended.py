"""Extended-precision (x87 80-bit, numpy.clongdouble) evaluation of the on-line stage -- TEST INFRASTRUCTURE ONLY.

SURVEY.md 8(c) "Parity metric", *also report, not gate*: entries above 1e-10 by the plain metric are adjudicated at
that omega by an 80-bit LU re-evaluation; an FP64 implementation passes there if its error against the 80-bit value
is <= a small multiple of the FP64 oracle's own error.  Used where the FP64 oracle itself is not accurate to 1e-10
(e.g. kappa(K) = 1e8, where two FP64 methods that do not share rounding differ by ~kappa u).

Same formulas and order as oracle/podp_oracle.py (P:593-596 eqn:ReducedA, P:600-604 eqn:podprealmpt,
P:606-620 eqn:podpimagmpt, P:632-661 lemma:certificate), carried in long double.  The solve is a textbook
Gaussian elimination with partial pivoting (|.| of the complex entry) written out, since LAPACK has no long double.
Pinned in tests/test_oracle_pins.py (agreement with the FP64 oracle on well-conditioned input, residual of the
solve in long double, r = 1 closed form).
"""
from __future__ import annotations

import numpy as np

from .podp_oracle import ENTRY_ORDER

LD = np.longdouble
CLD = np.clongdouble


def solve_ld(A, B):
    """X = A^{-1} B by Gaussian elimination with partial pivoting in complex long double (row interchanges on the
    largest |a_ik|, then forward elimination and back substitution)."""
    A = np.array(A, dtype=CLD)
    B = np.array(B, dtype=CLD)
    n = A.shape[0]
    for k in range(n):
        p = k + int(np.argmax(np.abs(A[k:, k])))
        if p != k:
            A[[k, p]] = A[[p, k]]
            B[[k, p]] = B[[p, k]]
        piv = A[k, k]
        for i in range(k + 1, n):
            l = A[i, k] / piv
            A[i, k:] -= l * A[k, k:]
            B[i] -= l * B[k]
    X = np.zeros_like(B)
    for k in range(n - 1, -1, -1):
        acc = B[k].copy()
        for j in range(k + 1, n):
            acc -= A[k, j] * X[j]
        X[k] = acc / A[k, k]
    return X


def evaluate_one_ld(ops, omega: float) -> dict:
    """R (omega-dependent part, PODP_FLAG_OUT_R convention), I and Delta at one omega in long double; returned as
    float64 6-vectors in ENTRY_ORDER (rounded once at the end)."""
    w = LD(omega)
    nu = LD(ops.nu)
    s = w * nu
    K = np.array(ops.K, dtype=CLD)
    M = np.array(ops.M, dtype=CLD)
    K_R = K if ops.K_R is None else np.array(ops.K_R, dtype=CLD)
    B = np.array(ops.b0, dtype=CLD) + w * np.array(ops.b1, dtype=CLD)
    P = solve_ld(K + CLD(1j) * s * M, B)
    a3 = LD(ops.alpha) ** 3
    S = np.array(ops.S, dtype=LD)
    H = np.array(ops.H, dtype=CLD)
    r = P.shape[0]
    Wt = np.zeros((6 + 2 * r, 3), dtype=CLD)
    for i in range(3):
        Wt[2 * i, i] = 1
        Wt[2 * i + 1, i] = w
        Wt[6:6 + r, i] = -P[:, i]
        Wt[6 + r:, i] = -CLD(1j) * s * P[:, i]
    G = np.array(ops.G, dtype=CLD)
    X = Wt.conj().T @ G @ Wt
    n = [max(LD(0), X[i, i].real) for i in range(3)]
    R6, I6, D6 = np.zeros(6), np.zeros(6), np.zeros(6)
    for e, (i, j) in enumerate(ENTRY_ORDER):
        R6[e] = float(-(a3 / 4) * (P[:, i].conj() @ (K_R @ P[:, j])).real)
        quad = P[:, i].conj() @ ((nu * M) @ P[:, j])
        lin = H[i] @ P[:, j] + H[j] @ P[:, i]
        I6[e] = float(w * a3 / 4 * (S[i, j] + (quad + lin).real))
        m = max(LD(0), n[i] + n[j] - 2 * X[i, j].real) if i != j else LD(0)
        D6[e] = float(a3 / (8 * LD(ops.alpha_lb)) * (n[i] + n[j] + m))
    return dict(R6=R6, I6=I6, D6=D6, P=P)
