"""Per-direction reduced bases (NEXT row N1 of SURVEY 8(f)): the paper's literal form, U_i^M per direction i with
M_i modes each, reduced systems A_i^M = (U_i^M)^H A U_i^M (eqn:ReducedA), cross blocks
K_ij^M = (U_i^M)^H K U_j^M (eqn:podprealmpt) and C_ij^M (eqn:podpimagmpt).

It is expressed exactly through the C ABI's shared-basis operands (include/podp.h, field M_I): with
U = [U_1 U_2 U_3] and r = M_1 + M_2 + M_3,
    K, M      block-diagonal  diag(K_11, K_22, K_33), diag(M_11, M_22, M_33)     (the three A_i^M solves)
    b0, b1    column i = (0, .., (U_i)^H B_i, .., 0)                            (r_i^M in block i only)
    K_R, M_I  the full block matrices [K_ij^M], [C_ij^M / nu]                   (the cross terms of R and I)
    H         row i = [h_i^(1), h_i^(2), h_i^(3)], h_i^(j) = o_i^T C2 U_j + t_i U_j
    G         Gram of [B0_1, B1_1, B0_2, B1_2, B0_3, B1_3 | K U | M U], placed from the direction Grams
              G_ij = W_i^H W_j, W_i = [B0_i, B1_i | K U_i | M U_i] (Lemma 4.1 fast form)
so that column i of P is (0, p_i^M, 0), p_i^H K_R p_j = p_i^H K_ij p_j, and the residual of column i is the
direction-i residual of Lemma 4.1.  The LU of a block-diagonal matrix with partial pivoting never leaves the
diagonal block (all other entries of the column are exact zeros), so the kernels solve the three systems exactly.
This module only places blocks (argument marshalling); every arithmetic step runs in libpodp.
"""
from __future__ import annotations

import numpy as np

from .adapt import ReducedOperators


def slot_map(m, i: int) -> np.ndarray:
    """Rows of the stacked (6 + 2r) factor that hold the columns of W_i = [B0_i, B1_i | K U_i | M U_i]."""
    off = np.concatenate([[0], np.cumsum(m)])
    r = int(off[-1])
    return np.concatenate([[2 * i, 2 * i + 1], 6 + np.arange(off[i], off[i + 1]),
                           6 + r + np.arange(off[i], off[i + 1])])


def embed(Kb, Mb, b0, b1, Hb, N0, S, Gx, nu: float, alpha: float, alpha_lb: float) -> ReducedOperators:
    """Kb[i][j], Mb[i][j]: M_i x M_j blocks (K_ij^M, C_ij^M / nu); b0[i], b1[i]: length-M_i vectors (r_i^M parts);
    Hb[i][j]: length-M_j row h_i^(j); Gx[i][j]: (2 + 2 M_i) x (2 + 2 M_j) direction Grams W_i^H W_j.
    Returns podp_create operands."""
    m = [int(np.asarray(b0[i]).shape[0]) for i in range(3)]
    off = np.concatenate([[0], np.cumsum(m)])
    r = int(off[-1])
    K = np.zeros((r, r), complex)
    M = np.zeros((r, r), complex)
    KR = np.zeros((r, r), complex)
    MI = np.zeros((r, r), complex)
    B0 = np.zeros((r, 3), complex)
    B1 = np.zeros((r, 3), complex)
    H = np.zeros((3, r), complex)
    for i in range(3):
        si = slice(off[i], off[i + 1])
        B0[si, i] = b0[i]
        B1[si, i] = b1[i]
        for j in range(3):
            sj = slice(off[j], off[j + 1])
            KR[si, sj] = Kb[i][j]
            MI[si, sj] = Mb[i][j]
            H[i, sj] = Hb[i][j]
        K[si, si] = Kb[i][i]
        M[si, si] = Mb[i][i]
    G = np.zeros((6 + 2 * r, 6 + 2 * r), complex)
    for i in range(3):
        for j in range(3):
            G[np.ix_(slot_map(m, i), slot_map(m, j))] = Gx[i][j]
    return ReducedOperators(K=K, M=M, b0=B0, b1=B1, N0=np.asarray(N0, float), S=np.asarray(S, float), H=H,
                            G=G, nu=float(nu), alpha=float(alpha), alpha_lb=float(alpha_lb),
                            K_R=KR, M_I=MI)


def split_P(P, m) -> list:
    """Column i of the embedded P (3 x r, as returned with want_P) -> p_i^M (length M_i)."""
    off = np.concatenate([[0], np.cumsum(m)])
    return [P[..., i, off[i]:off[i + 1]] for i in range(3)]
