"""Per-direction PODP, the paper's literal form (NEXT row N1) -- TEST INFRASTRUCTURE ONLY (oracle/__init__.py).

Each direction i has its own TSVD basis U_i (N x M_i) and reduced system
    A_i^M[omega] p_i = r_i^M[omega],  A_i^M = U_i^H (K + i omega nu M) U_i,  r_i^M = U_i^H (B0_i + omega B1_i)
(eqn:ReducedA, BASELINE sign), and the MPT couples directions through the cross blocks
    R_ij = -(alpha^3/4) Re(p_i^H K_ij p_j),  K_ij = U_i^H K U_j                          (eqn:podprealmpt)
    I_ij = (omega alpha^3/4) (S_ij + Re(p_i^H C_ij p_j + h_i^(j) p_j + h_j^(i) p_i)),
           C_ij = U_i^H C U_j,  h_i^(j) = o_i^T C2 U_j + t_i U_j   (here v_i^T C U_j)     (eqn:podpimagmpt)
The certificate uses the direction-i residual r_i = B0_i + omega B1_i - (K + i omega nu M) U_i p_i, written as
W_i w_i with W_i = [B0_i, B1_i | K U_i | M U_i] and w_i = (1, omega, -p_i, -i omega nu p_i), so that
X_ij = r_i^H r_j = w_i^H (W_i^H W_j) w_j (Lemma 4.1 fast form).  Written directly from these
definitions: nothing here uses the block embedding the CUDA path is fed with.
"""
from __future__ import annotations

import numpy as np

from .podp_oracle import to6


def tsvd_per_direction(Q_list, tol_sigma: float):
    """D_i = [q_i[omega_1], ..., q_i[omega_N]] and its TSVD (Algorithm 1 lines 5-6), i = 1, 2, 3.
    Q_list: snapshots, each N x 3.  Returns [U_1, U_2, U_3]."""
    Us = []
    for i in range(3):
        D = np.stack([q[:, i] for q in Q_list], axis=1)
        U, s, _ = np.linalg.svd(D, full_matrices=False)
        Us.append(U[:, :int(np.sum(s / s[0] >= tol_sigma))])
    return Us


class PerDirectionROM:
    """Cross blocks of the per-direction reduced model built from a full-order system `fom` and bases Us."""

    def __init__(self, fom, Us):
        self.Us = Us
        self.nu, self.alpha, self.alpha_lb = fom.nu, fom.alpha, fom.alpha_lb
        K, M, C, v = fom.K_full, fom.M_full, fom.C_full, fom.v
        self.K = [[Us[i].conj().T @ K @ Us[j] for j in range(3)] for i in range(3)]
        self.Mm = [[Us[i].conj().T @ M @ Us[j] for j in range(3)] for i in range(3)]
        self.C = [[Us[i].conj().T @ C @ Us[j] for j in range(3)] for i in range(3)]
        self.h = [[v[:, i] @ C @ Us[j] for j in range(3)] for i in range(3)]
        self.S = np.real(v.T @ C @ v)
        self.b0 = [Us[i].conj().T @ fom.B0f[:, i] for i in range(3)]
        self.b1 = [Us[i].conj().T @ fom.B1f[:, i] for i in range(3)]
        W = [np.column_stack([fom.B0f[:, i], fom.B1f[:, i], K @ Us[i], M @ Us[i]]) for i in range(3)]
        self.Gx = [[W[i].conj().T @ W[j] for j in range(3)] for i in range(3)]
        self.N0 = np.eye(3)

    def evaluate_one(self, omega: float, out_R: bool = False) -> dict:
        a3 = self.alpha ** 3
        s = omega * self.nu
        p = [np.linalg.solve(self.K[i][i] + 1j * s * self.Mm[i][i], self.b0[i] + omega * self.b1[i])
             for i in range(3)]
        R = np.zeros((3, 3))
        I = np.zeros((3, 3))
        for i in range(3):
            for j in range(3):
                R[i, j] = -(a3 / 4.0) * np.real(np.vdot(p[i], self.K[i][j] @ p[j]))
                I[i, j] = omega * a3 / 4.0 * (self.S[i, j] + np.real(np.vdot(p[i], self.C[i][j] @ p[j])
                                                                    + self.h[i][j] @ p[j] + self.h[j][i] @ p[i]))
        w = [np.concatenate([[1.0, omega], -p[i], -1j * s * p[i]]) for i in range(3)]
        X = np.array([[np.vdot(w[i], self.Gx[i][j] @ w[j]) for j in range(3)] for i in range(3)])
        n = np.array([max(0.0, float(np.real(X[i, i]))) for i in range(3)])
        D = np.zeros((3, 3))
        for i in range(3):
            for j in range(3):
                m = max(0.0, n[i] + n[j] - 2.0 * float(np.real(X[i, j]))) if i != j else 0.0
                D[i, j] = a3 / (8.0 * self.alpha_lb) * (n[i] + n[j] + m)
        T1 = R if out_R else self.N0 + R
        return dict(p=p, T1=T1, R=R, I=I, Delta=D, n=n)

    def evaluate(self, omegas, out_R: bool = False):
        """F x 6 (T1, I, Delta) in ENTRY_ORDER."""
        T1 = np.zeros((len(omegas), 6))
        I = np.zeros_like(T1)
        D = np.zeros_like(T1)
        for f, w in enumerate(omegas):
            o = self.evaluate_one(float(w), out_R)
            T1[f], I[f], D[f] = to6(o["T1"]), to6(o["I"]), to6(o["Delta"])
        return T1, I, D
