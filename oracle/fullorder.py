"""Full-order formulas used only to PIN the reduced oracle (TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py).

These are the paper's Full Matrix Method (FMM) expressions evaluated on the reconstructed full-order field
q_i = U p_i (eqn:solution:rebreakdown), with the tiny synthetic full-order system of config 0.
"""
from __future__ import annotations

import numpy as np


def reconstruct(U, P):
    """q_i^PODP = U^M p_i^M."""
    return U @ P


def fmm_R(Q, K_full, alpha: float):
    """R_ij = -(alpha^3/4) conj(q_i)^T K q_j (eqn:Rmatrixmeth); real part."""
    R = np.zeros((3, 3))
    for i in range(3):
        for j in range(3):
            R[i, j] = -(alpha ** 3 / 4.0) * np.real(np.vdot(Q[:, i], K_full @ Q[:, j]))
    return R


def fmm_I(Q, v, C_full, alpha: float, omega: float):
    """I_ij from the Gram form of eqn:Itensor with Remark 3.1's shared discretisation:
    I_ij = (omega alpha^3 / 4) Re( (q_i + v_i)^H C (q_j + v_j) ),  C = nu-weighted conductor matrix, v real."""
    I = np.zeros((3, 3))
    for i in range(3):
        for j in range(3):
            a = Q[:, i] + v[:, i]
            b = Q[:, j] + v[:, j]
            I[i, j] = omega * alpha ** 3 / 4.0 * np.real(np.vdot(a, C_full @ b))
    return I


def full_residual(K_full, M_full, B0f, B1f, U, P, nu: float, omega: float):
    """Explicit full-order residual r_i = B0f_i + omega B1f_i - (K + i omega nu M) U p_i (P:480-483 with the BASELINE
    sign, reading U1).  Returns N x 3."""
    s = omega * nu
    Q = U @ P
    return (B0f + omega * B1f) - (K_full @ Q + 1j * s * (M_full @ Q))


def full_solve(K_full, M_full, B0f, B1f, nu: float, omega: float):
    """Full-order solve A[omega] q = r (eqn:Linear), dense LAPACK."""
    return np.linalg.solve(K_full + 1j * omega * nu * M_full, B0f + omega * B1f)
