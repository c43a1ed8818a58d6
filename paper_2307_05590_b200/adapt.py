"""Algorithm 1 driver (alg:adapt) around the on-line path -- NEXT row N2 of SURVEY 8(f).

Off-line stage (lines 3-6, 16-19) on the GPU through library calls: the dense full-order snapshot solves of
eqn:Linear are batched cuSOLVER LU solves (torch.linalg.solve), the TSVD of D is a cuSOLVER SVD,
and the Galerkin projections plus the residual Gram G = W^H W of Lemma 4.1 are cuBLAS
products.  The reduced operators are then packed by podp_create and the certification + greedy step
(lines 10-15) run in this package's own kernels (podp_eval, podp_select).  There is no CPU path: a missing CUDA
device or libpodp.so raises.

Readings (N2): one shared basis, the TSVD of D = [D_1 D_2 D_3] (reading U3); s_k kept when
s_k / s_1 >= TOL_Sigma (P:584 garbled); the first certification runs before the loop test so that line 8 has a
Lambda; |B_alpha| is the caller's `vol`; the adaption window is the output grid the caller passes (P:997 adapts on
[1e1, 1e7] with snapshots on [1e1, 1e8]).
"""
from __future__ import annotations

import dataclasses
import math
import time

import numpy as np

from .podp import Evaluator


@dataclasses.dataclass
class ReducedOperators:
    """podp_create inputs (see include/podp.h podp_operators)."""
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
    M_I: np.ndarray | None = None

    @property
    def r(self) -> int:
        return int(self.K.shape[0])


def log_snapshots(n0: int, lo: float = 1e1, hi: float = 1e8) -> np.ndarray:
    """Line 3: initial log-spaced snapshot frequencies (N = 13 on [1e1, 1e8] rad/s)."""
    return np.logspace(math.log10(lo), math.log10(hi), n0)


class FullOrderGPU:
    """Device-resident full-order system (K_full, M_full complex N x N; B0f, B1f complex N x 3; v real N x 3)."""

    def __init__(self, fom, device: int = 0):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("adapt: a CUDA device is required (no CPU path)")
        self.dev = torch.device("cuda", device)
        c = lambda x: torch.as_tensor(np.asarray(x, dtype=np.complex128), device=self.dev)  # noqa: E731
        self.K, self.M = c(fom.K_full), c(fom.M_full)
        self.B0, self.B1 = c(fom.B0f), c(fom.B1f)
        self.v = c(fom.v)                     # real coefficients, held complex for the products
        self.nu, self.alpha, self.alpha_lb = float(fom.nu), float(fom.alpha), float(fom.alpha_lb)
        self.N = int(self.K.shape[0])

    def solve(self, omegas) -> "torch.Tensor":  # noqa: F821
        """Lines 4 / 16: q_i[omega] for every omega, one batched LU solve.  Returns (n, N, 3)."""
        import torch
        w = torch.as_tensor(np.asarray(omegas, dtype=np.float64), device=self.dev).to(torch.complex128)
        A = self.K.unsqueeze(0) + (1j * self.nu) * w.view(-1, 1, 1) * self.M.unsqueeze(0)
        B = self.B0.unsqueeze(0) + w.view(-1, 1, 1) * self.B1.unsqueeze(0)
        return torch.linalg.solve(A, B)

    def reduce(self, U) -> ReducedOperators:
        """Galerkin projection onto U (N x r) and the Gram of W = [B0_1, B1_1, B0_2, B1_2, B0_3, B1_3 | K U | M U]."""
        import torch
        Uh = U.conj().transpose(0, 1)
        KU, MU = self.K @ U, self.M @ U
        K, M = Uh @ KU, Uh @ MU
        W = torch.cat([torch.stack([self.B0, self.B1], dim=2).reshape(self.N, 6), KU, MU], dim=1)
        G = W.conj().transpose(0, 1) @ W
        C = self.nu * self.M
        vt = self.v.transpose(0, 1)
        S = (vt @ C @ self.v).real
        H = vt @ C @ U
        herm = lambda X: 0.5 * (X + X.conj().transpose(0, 1))  # noqa: E731
        h = lambda X: X.cpu().numpy()  # noqa: E731
        return ReducedOperators(K=h(herm(K)), M=h(herm(M)), b0=h(Uh @ self.B0), b1=h(Uh @ self.B1), N0=np.eye(3),
                                S=h(0.5 * (S + S.transpose(0, 1))), H=h(H), G=h(herm(G)), nu=self.nu,
                                alpha=self.alpha, alpha_lb=self.alpha_lb)


    def reduce_per_direction(self, Us) -> ReducedOperators:
        """NEXT row N1: per-direction bases U_i (N x M_i) in the block embedding of perdir.py: U = [U_1 U_2 U_3],
        K, M block-diagonal (the three A_i^M), K_R = [K_ij^M], M_I = [C_ij^M]/nu, b column i
        restricted to block i; G is then the Gram of [B0_1, B1_1, ... | K U | M U] as in the shared form."""
        import torch
        m = [int(U.shape[1]) for U in Us]
        U = torch.cat(list(Us), dim=1)
        full = self.reduce(U)
        off = np.concatenate([[0], np.cumsum(m)])
        blk = np.zeros((full.r, full.r), dtype=bool)
        rows = np.zeros((full.r, 3), dtype=bool)
        for i in range(3):
            blk[off[i]:off[i + 1], off[i]:off[i + 1]] = True
            rows[off[i]:off[i + 1], i] = True
        return dataclasses.replace(full, K=np.where(blk, full.K, 0), M=np.where(blk, full.M, 0), K_R=full.K,
                                   M_I=full.M, b0=np.where(rows, full.b0, 0), b1=np.where(rows, full.b1, 0))


def tsvd(D, tol_sigma: float):
    """Lines 6 / 19: D^M = U^M Sigma^M (V^M)^H, keeping s_k / s_1 >= TOL_Sigma."""
    import torch
    U, s, _ = torch.linalg.svd(D, full_matrices=False)
    M = int((s / s[0] >= tol_sigma).sum().item())
    return U[:, :M]


def run_adaptive(fom, omegas, n0: int = 13, n_star: int = 2, tol_sigma: float = 1e-6, tol_delta: float = 1e-3,
                 max_k: int = 4, vol: float = 1.0, theta: float | None = None, snap0=None, device: int = 0,
                 flags: int = 0, per_direction: bool = False):
    """Algorithm 1 lines 1-26 with the certification on `omegas` (the output grid / adaption window).

    Returns (ops, outputs dict(T1, I, Delta) of the final ROM on omegas (device tensors, n_obj = 1), history) where
    history[k-1] = dict(k, N, r, Lambda, snap, new, t_offline, t_online) -- times in seconds, host clock around
    synchronised phases."""
    import torch
    g = fom if isinstance(fom, FullOrderGPU) else FullOrderGPU(fom, device)
    om = torch.as_tensor(np.asarray(omegas, dtype=np.float64), device=g.dev)
    snap = [float(w) for w in (log_snapshots(n0) if snap0 is None else snap0)]          # line 3
    Q = dict(zip(snap, g.solve(snap).unbind(0)))                                          # line 4
    k = 1
    history = []
    t0 = time.perf_counter()
    while True:
        if per_direction:                                                                 # N1: D_i, U_i^M
            Us = [tsvd(torch.stack([Q[w][:, i] for w in snap], dim=1), tol_sigma) for i in range(3)]
            ops = g.reduce_per_direction(Us)
            m = [int(U.shape[1]) for U in Us]
        else:
            D = torch.cat([Q[w] for w in snap], dim=1)                                    # lines 5 / 18
            U = tsvd(D, tol_sigma)                                                        # lines 6 / 19
            ops = g.reduce(U)
            m = [ops.r]
        torch.cuda.synchronize(g.dev)
        t1 = time.perf_counter()
        ev = Evaluator(ops, device=g.dev.index)
        out = ev.eval(om, flags=flags)                                                    # line 11
        new, _idx, Lam, _lam = ev.select(om, out["Delta"][0], snap, n_star,
                                         0.0 if theta is None else theta)                 # lines 12-15
        ev.close()
        t2 = time.perf_counter()
        rec = dict(k=k, N=len(snap), r=ops.r, m=m, Lambda=float(Lam), snap=list(snap), new=[], t_offline=t1 - t0,
                   t_online=t2 - t1)
        history.append(rec)
        if not (Lam / vol > tol_delta and k < max_k):                                     # line 8
            return ops, out, history
        k += 1                                                                            # line 9
        t0 = time.perf_counter()
        new = [float(w) for w in new]
        rec["new"] = list(new)
        Q.update(zip(new, g.solve(new).unbind(0)))                                        # line 16
        snap = sorted(snap + new)                                                         # line 17
