"""NEXT row N2: Algorithm 1 (alg:adapt) on the synthetic full-order system of make_fullorder.

CPU part pins the oracle driver (oracle/adapt.py) to the full-order problem it reduces; the GPU part runs the
product driver (paper_2307_05590_b200.adapt: cuSOLVER/cuBLAS off-line stage + this package's eval/select kernels)
and compares every decision and output with the oracle driver."""
import math

import numpy as np
import pytest

import oracle
from oracle import adapt as oadapt
from oracle.fullorder import fmm_I, fmm_R, full_residual
from podp_inputs import generators as g

OMEGA = g.omega_grid(401, 1e1, 1e7)     # adaption window [1e1, 1e7], snapshots on [1e1, 1e8]


@pytest.fixture(scope="module")
def fom():
    return g.make_fullorder()


@pytest.fixture(scope="module")
def vol(fom):
    return fom.alpha ** 3 * 4.0 * math.pi / 3.0   # |B_alpha| for the unit ball scaled by alpha (reading, DESIGN 3)


@pytest.fixture(scope="module")
def run4(fom, vol):
    return oadapt.run_adaptive(fom, OMEGA, tol_delta=1e-12, max_k=4, vol=vol)


def test_N2_oracle_snapshot_sequence(run4):
    # P:834 / P:897: iterations k = 1..4 give N = 13, 15, 17, 19 with N* = 2, at most one per interval
    _ops, _out, h = run4
    assert [x["N"] for x in h] == [13, 15, 17, 19] and [x["k"] for x in h] == [1, 2, 3, 4]
    for a, b in zip(h[:-1], h[1:]):
        assert len(a["new"]) == 2 and all(w in OMEGA for w in a["new"]) and not set(a["new"]) & set(a["snap"])
        assert b["snap"] == sorted(a["snap"] + a["new"])
        # at most one new snapshot per interval
        pos = [np.searchsorted(a["snap"], w) for w in a["new"]]
        assert len(set(pos)) == len(pos)


def test_N2_oracle_stop_rules(fom, vol):
    # line 8: a huge TOL_Delta stops after the initial certification (k = 1, N unchanged)
    _o, _x, h = oadapt.run_adaptive(fom, OMEGA, tol_delta=1e30, max_k=10, vol=vol)
    assert len(h) == 1 and h[0]["N"] == 13 and h[0]["new"] == []
    # theta-threshold variant with theta = 1: only the global-max interval is refined each iteration
    _o, _x, h = oadapt.run_adaptive(fom, OMEGA, tol_delta=1e-12, max_k=3, vol=vol, theta=1.0)
    assert [x["N"] for x in h] == [13, 14, 15]


def test_N2_oracle_rom_reproduces_snapshots(fom, run4):
    # the POD space contains every snapshot up to TOL_Sigma, so the reduced solve reproduces q at snapshot omegas
    ops, _out, h = run4
    U = oadapt.tsvd(np.concatenate([oadapt.full_solve(fom, w) for w in h[-1]["snap"]], axis=1), 1e-6)
    for w in h[-1]["snap"][::3]:
        P = oracle.solve_reduced(ops.K, ops.M, ops.b0, ops.b1, ops.nu, w)
        q = oadapt.full_solve(fom, w)
        assert np.linalg.norm(U @ P - q) <= 1e-5 * np.linalg.norm(q)


def test_N2_oracle_reduced_forms_match_full_order(fom, run4):
    # R, I of the reduced formulas equal the FMM formulas on q = U p, and the Gram-form certificate's
    # n_i equals |r_i|^2 of the explicit full-order residual (Lemma 4.1)
    ops, _out, h = run4
    U = oadapt.tsvd(np.concatenate([oadapt.full_solve(fom, w) for w in h[-1]["snap"]], axis=1), 1e-6)
    for w in (37.0, 2.1e3, 4.4e5, 6.0e6):
        o = oracle.evaluate_one(ops, w, out_R=True)
        Q = U @ o["P"]
        Rf = fmm_R(Q, fom.K_full, fom.alpha)
        If = fmm_I(Q, fom.v, fom.C_full, fom.alpha, w)
        assert np.max(np.abs(o["R"] - Rf)) <= 1e-9 * np.max(np.abs(Rf))
        assert np.max(np.abs(o["I"] - If)) <= 1e-9 * np.max(np.abs(If))
        _D, n, _X = oracle.certificate(o["P"], ops.G, ops.nu, w, ops.alpha, ops.alpha_lb)
        r = full_residual(fom.K_full, fom.M_full, fom.B0f, fom.B1f, U, o["P"], fom.nu, w)
        nex = np.real(np.sum(r.conj() * r, axis=0))
        scale = np.linalg.norm(fom.B0f + w * fom.B1f, axis=0) ** 2     # cancellation floor of the Gram form
        assert np.all(np.abs(n - nex) <= 1e-12 * scale)


def test_N2_oracle_certificate_decreases(run4, vol):
    # P:834-838 (Figs. 5-6): the adaptive snapshots reduce Lambda; for this recipe by > 2 orders over k = 1..4
    h = run4[2]
    lam = [x["Lambda"] / vol for x in h]
    assert lam[-1] < 1e-2 * lam[0] and all(b < a for a, b in zip(lam[:-1], lam[1:]))


def _per_entry_parity(ops, out):
    """Per-entry gates of SURVEY 8(c) (1e-10 x term magnitude on R and I, 1e-8 on Delta) between the GPU driver's
    final on-line outputs and the oracle evaluated on the SAME reduced operators (the off-line stages of the two
    drivers round differently, so their ROMs differ at the TSVD-truncation level; the decisions are compared
    separately), plus Lambda of the selection against the oracle's brute-force select on the oracle's Delta."""
    import dataclasses
    from oracle.parity import TOL_DELTA, TOL_RI, magnitudes
    from oracle.podp_oracle import certificate, mpt_I, mpt_R, solve_reduced
    T1, I, D = (out[k][0].cpu().numpy() for k in ("T1", "I", "Delta"))
    M_I = ops.M if getattr(ops, "M_I", None) is None else ops.M_I      # N1 embedding: I uses the cross blocks
    K_R = ops.K if ops.K_R is None else ops.K_R
    ops_m = dataclasses.replace(ops, M=M_I)                             # magnitudes' ||p||_M in the I metric
    worst = np.zeros(3)
    oD = np.zeros((len(OMEGA), 6))
    for f, w in enumerate(OMEGA):
        w = float(w)
        P = solve_reduced(ops.K, ops.M, ops.b0, ops.b1, ops.nu, w)
        oD[f] = oracle.to6(certificate(P, ops.G, ops.nu, w, ops.alpha, ops.alpha_lb)[0])
        if f % 5:
            continue
        oR = oracle.to6(mpt_R(P, K_R, ops.alpha))
        oI = oracle.to6(mpt_I(P, M_I, ops.S, ops.H, ops.nu, ops.alpha, w))
        magR, magI, magD = magnitudes(ops_m, w, P)
        e = (np.abs(T1[f] - oR) / magR, np.abs(I[f] - oI) / magI,
             np.abs(D[f] - oD[f]) / np.maximum(oD[f], 1e-6 * magD))
        worst = np.maximum(worst, [x.max() for x in e])
    assert worst[0] <= TOL_RI and worst[1] <= TOL_RI and worst[2] <= TOL_DELTA, worst
    return oD


def _check_lambda(ops, oD, rec):
    """Lambda of the final certification: GPU select vs the oracle's select on the oracle's Delta of the same ROM,
    under the Delta gate at the maximising entry (1e-8 x max(Delta, 1e-6 mag^Delta): near-zero residuals are
    cancellation-limited)."""
    from oracle.parity import TOL_DELTA, magnitudes
    oLam = oracle.select(OMEGA, oD, rec["snap"], 2)[2]
    f, e = np.argwhere(oD == oLam)[0]
    magD = magnitudes(ops, float(OMEGA[f]))[2][e]
    assert abs(rec["Lambda"] - oLam) <= TOL_DELTA * max(oLam, 1e-6 * magD)


@pytest.mark.gpu
def test_N2_gpu_driver_matches_oracle(torch_cuda, fom, vol, run4):
    from paper_2307_05590_b200 import FLAG_OUT_R, adapt
    ops, out, h = adapt.run_adaptive(fom, OMEGA, tol_delta=1e-12, max_k=4, vol=vol, flags=FLAG_OUT_R)
    o_ops, (oT1, oI, oD), oh = run4
    assert [x["N"] for x in h] == [x["N"] for x in oh]
    assert [x["r"] for x in h] == [x["r"] for x in oh]
    for a, b in zip(h, oh):
        assert a["snap"] == b["snap"] and a["new"] == b["new"]        # every greedy decision identical
        assert abs(a["Lambda"] - b["Lambda"]) <= 1e-2 * b["Lambda"]   # different ROMs (off-line rounding)
    oD_same = _per_entry_parity(ops, out)
    _check_lambda(ops, oD_same, h[-1])


def test_N2_oracle_per_direction_runs(fom, vol):
    # N1 inside Algorithm 1: per-direction TSVDs (lines 6/19 for i = 1, 2, 3); same snapshot bookkeeping
    _o, _x, h = oadapt.run_adaptive(fom, OMEGA, tol_delta=1e-12, max_k=3, vol=vol, per_direction=True)
    assert [x["N"] for x in h] == [13, 15, 17] and all(len(x["m"]) == 3 for x in h)
    assert h[-1]["Lambda"] < h[0]["Lambda"]


@pytest.mark.gpu
def test_N2_gpu_driver_per_direction_matches_oracle(torch_cuda, fom, vol):
    from paper_2307_05590_b200 import FLAG_OUT_R, adapt
    ops, out, h = adapt.run_adaptive(fom, OMEGA, tol_delta=1e-12, max_k=3, vol=vol, per_direction=True,
                                     flags=FLAG_OUT_R)
    _o, _x, oh = oadapt.run_adaptive(fom, OMEGA, tol_delta=1e-12, max_k=3, vol=vol, per_direction=True)
    for a, b in zip(h, oh):
        assert a["m"] == b["m"] and a["snap"] == b["snap"] and a["new"] == b["new"]
        assert abs(a["Lambda"] - b["Lambda"]) <= 1e-2 * b["Lambda"]
    oD_same = _per_entry_parity(ops, out)
    _check_lambda(ops, oD_same, h[-1])
