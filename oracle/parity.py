"""Parity metric of SURVEY.md 8(c) (reading U17) -- TEST INFRASTRUCTURE ONLY.

Per-entry term magnitudes computed from the oracle's own quantities:
  mag^R_ij = (alpha^3/4) ||p_i||_K ||p_j||_K               (K_R positive definite; else ||p_i|| ||K_R||_2 ||p_j||)
  mag^I_ij = (|omega| alpha^3/4)(|S_ij| + nu ||p_i||_M ||p_j||_M + |h_i p_j| + |h_j p_i|)
  mag^D_ij = (alpha^3/(4 alpha_LB)) (Mw_ii + Mw_jj + Mw_ij),  Mw_ij = |w_i|^T |G| |w_j|
Gates: |gpu - ora| <= 1e-10 mag (R, I);  |gpu - ora| <= 1e-8 max(Delta_ora, 1e-6 mag^D) (Delta).
"""
from __future__ import annotations

import numpy as np

from .podp_oracle import ENTRY_ORDER, residual_coeffs, solve_reduced

TOL_RI = 1e-10
TOL_DELTA = 1e-8


def magnitudes(ops, omega: float, P=None):
    if P is None:
        P = solve_reduced(ops.K, ops.M, ops.b0, ops.b1, ops.nu, omega)
    K_R = ops.K if ops.K_R is None else ops.K_R
    a3 = ops.alpha ** 3
    evK = np.linalg.eigvalsh(K_R)
    if evK[0] > 0:
        nK = np.array([np.sqrt(max(0.0, np.real(np.vdot(P[:, i], K_R @ P[:, i])))) for i in range(3)])
        kfac = 1.0
    else:
        nK = np.linalg.norm(P, axis=0)
        kfac = float(np.max(np.abs(evK)))
    nM = np.array([np.sqrt(max(0.0, np.real(np.vdot(P[:, i], ops.M @ P[:, i])))) for i in range(3)])
    Wt = residual_coeffs(P, ops.nu, omega)
    aW = np.abs(Wt)
    aG = np.abs(ops.G)
    Mw = aW.T @ aG @ aW
    magR = np.zeros(6)
    magI = np.zeros(6)
    magD = np.zeros(6)
    for e, (i, j) in enumerate(ENTRY_ORDER):
        magR[e] = a3 / 4.0 * kfac * nK[i] * nK[j]
        magI[e] = abs(omega) * a3 / 4.0 * (abs(ops.S[i, j]) + ops.nu * nM[i] * nM[j]
                                          + abs(np.dot(ops.H[i], P[:, j])) + abs(np.dot(ops.H[j], P[:, i])))
        magD[e] = a3 / (4.0 * ops.alpha_lb) * (Mw[i, i] + Mw[j, j] + Mw[i, j])
    return magR, magI, magD


def errors(ops, omega: float, gpu_R6, gpu_I6, gpu_D6, ora_R6, ora_I6, ora_D6):
    """Return (eR, eI, eD) per-entry normalised errors; each must be <= 1 to pass (eR, eI scaled by TOL_RI,
    eD by TOL_DELTA)."""
    magR, magI, magD = magnitudes(ops, omega)
    eR = np.abs(np.asarray(gpu_R6) - ora_R6) / np.maximum(magR, 1e-300)
    eI = np.abs(np.asarray(gpu_I6) - ora_I6) / np.maximum(magI, 1e-300)
    eD = np.abs(np.asarray(gpu_D6) - ora_D6) / np.maximum(np.maximum(ora_D6, 1e-6 * magD), 1e-300)
    return eR, eI, eD
