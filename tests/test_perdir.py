"""NEXT row N1: per-direction reduced bases (the paper's literal U_i^M form).

CPU: the literal per-direction oracle (oracle/perdir.py) is pinned to (a) the shared-basis oracle when the three
bases coincide, (b) the full-order FMM formulas and explicit residuals on q_i = U_i p_i, (c) the snapshots it was
built from; and the block embedding of paper_2307_05590_b200.perdir fed to the shared-basis oracle reproduces it.
GPU: the embedding evaluated by libpodp (M_I operand) matches the literal oracle."""
import numpy as np
import pytest

import oracle
from oracle import adapt as oadapt
from oracle.fullorder import fmm_I, fmm_R
from oracle.parity import TOL_DELTA, TOL_RI, errors
from oracle.perdir import PerDirectionROM, tsvd_per_direction
from podp_inputs import generators as g

W_TEST = (23.0, 911.0, 3.3e4, 1.7e6, 4.2e7)


@pytest.fixture(scope="module")
def fom():
    return g.make_fullorder()


@pytest.fixture(scope="module")
def snaps(fom):
    w = list(g.snapshot_grid(13))
    return w, [oadapt.full_solve(fom, x) for x in w]


@pytest.fixture(scope="module")
def rom(fom, snaps):
    return PerDirectionROM(fom, tsvd_per_direction(snaps[1], 1e-6))


def embedded(rom):
    from paper_2307_05590_b200 import perdir
    return perdir.embed(rom.K, [[rom.C[i][j] / rom.nu for j in range(3)] for i in range(3)], rom.b0, rom.b1,
                        rom.h, rom.N0, rom.S, rom.Gx, rom.nu, rom.alpha, rom.alpha_lb)


def test_N1_bases_differ(rom):
    m = [U.shape[1] for U in rom.Us]
    assert len(set(m)) >= 1 and all(1 <= x <= 13 for x in m)
    # the three direction subspaces are genuinely different (otherwise N1 would reduce to the shared form)
    s = np.linalg.svd(rom.Us[0].conj().T @ rom.Us[1], compute_uv=False)
    assert s.min() < 0.99


def test_N1_equal_bases_reduce_to_shared(fom, snaps):
    U = oadapt.tsvd(np.concatenate(snaps[1], axis=1), 1e-6)
    per = PerDirectionROM(fom, [U, U, U])
    sh = oadapt.reduced_operators(fom, U)
    for w in W_TEST:
        a = per.evaluate_one(w)
        b = oracle.evaluate_one(sh, w)
        eR, eI, eD = errors(sh, w, *(oracle.to6(a[k]) for k in ("T1", "I", "Delta")),
                            *(oracle.to6(b[k]) for k in ("T1", "I", "Delta")))
        assert eR.max() <= TOL_RI and eI.max() <= TOL_RI and eD.max() <= TOL_DELTA


def test_N1_full_order_pins(fom, rom):
    from oracle.fullorder import full_residual
    for w in W_TEST:
        o = rom.evaluate_one(w, out_R=True)
        Q = np.column_stack([rom.Us[i] @ o["p"][i] for i in range(3)])
        Rf, If = fmm_R(Q, fom.K_full, fom.alpha), fmm_I(Q, fom.v, fom.C_full, fom.alpha, w)
        assert np.max(np.abs(o["R"] - Rf)) <= 1e-9 * np.abs(Rf).max()
        assert np.max(np.abs(o["I"] - If)) <= 1e-9 * np.abs(If).max()
        for i in range(3):
            P = np.zeros((rom.Us[i].shape[1], 3), complex)
            P[:, i] = o["p"][i]
            r = full_residual(fom.K_full, fom.M_full, fom.B0f, fom.B1f, rom.Us[i], P, fom.nu, w)[:, i]
            scale = np.linalg.norm(fom.B0f[:, i] + w * fom.B1f[:, i]) ** 2
            assert abs(o["n"][i] - np.vdot(r, r).real) <= 1e-12 * scale


def test_N1_reproduces_snapshots(fom, snaps, rom):
    for w, q in list(zip(*snaps))[::4]:
        o = rom.evaluate_one(w)
        for i in range(3):
            assert np.linalg.norm(rom.Us[i] @ o["p"][i] - q[:, i]) <= 1e-5 * np.linalg.norm(q[:, i])


def test_N1_embedding_is_exact(rom):
    ops = embedded(rom)
    for w in W_TEST:
        a = rom.evaluate_one(w)
        P = oracle.solve_reduced(ops.K, ops.M, ops.b0, ops.b1, ops.nu, w)
        R = oracle.mpt_R(P, ops.K_R, ops.alpha)
        I = oracle.mpt_I(P, ops.M_I, ops.S, ops.H, ops.nu, ops.alpha, w)
        D, _, _ = oracle.certificate(P, ops.G, ops.nu, w, ops.alpha, ops.alpha_lb)
        eR, eI, eD = errors(ops, w, oracle.to6(np.eye(3) + R), oracle.to6(I), oracle.to6(D),
                            *(oracle.to6(a[k]) for k in ("T1", "I", "Delta")))
        assert eR.max() <= TOL_RI and eI.max() <= TOL_RI and eD.max() <= TOL_DELTA


@pytest.mark.gpu
def test_N1_gpu_parity(torch_cuda, rom):
    torch = torch_cuda
    from paper_2307_05590_b200 import Evaluator, FLAG_OUT_R, FLAG_PENCIL
    ops = embedded(rom)
    omega = g.omega_grid(257)
    ora = rom.evaluate(omega, out_R=True)
    for flags in (FLAG_OUT_R, FLAG_OUT_R | FLAG_PENCIL):
        ev = Evaluator(ops)
        out = ev.eval(torch.tensor(omega, device="cuda"), flags=flags)
        T1, I, D = (out[k][0].cpu().numpy() for k in ("T1", "I", "Delta"))
        assert (out["info"] == 0).all()
        worst = np.zeros(3)
        for f in range(0, len(omega), 8):
            eR, eI, eD = errors(ops, omega[f], T1[f], I[f], D[f], ora[0][f], ora[1][f], ora[2][f])
            worst = np.maximum(worst, [eR.max() / TOL_RI, eI.max() / TOL_RI, eD.max() / TOL_DELTA])
        assert (worst <= 1.0).all(), (flags, worst)
        ev.close()


@pytest.mark.gpu
def test_N1_literal_gpu_parity(torch_cuda, rom):
    """N1 in the paper's literal form (podp_create_perdir): three LU solves of sizes M_1, M_2, M_3 per omega
    (P:596), the cross-block contractions and the direction-Gram certificate, per entry
    against the literal oracle (oracle/perdir.py), with every LU kernel the library has for the padded max M_i;
    P column i equals (0, p_i, 0); a non-finite omega gives info -1 and NaN rows."""
    torch = torch_cuda
    from paper_2307_05590_b200 import (Evaluator, FLAG_LU_BLK, FLAG_LU_DYN, FLAG_LU_GENERIC, FLAG_LU_LL,
                                       FLAG_OUT_R, FLAG_PENCIL, PodpError)
    m = [U.shape[1] for U in rom.Us]
    ops = embedded(rom)                                  # only for the parity metric's magnitudes
    ev = Evaluator.per_direction(rom.K, [[rom.C[i][j] / rom.nu for j in range(3)] for i in range(3)], rom.b0,
                                 rom.b1, rom.h, rom.N0, rom.S, rom.Gx, rom.nu, rom.alpha, rom.alpha_lb)
    assert ev.r == sum(m) and ev.n_obj == 1
    omega = g.omega_grid(129)
    ora = rom.evaluate(omega, out_R=True)
    off = np.concatenate([[0], np.cumsum(m)])
    for fl in (0, FLAG_LU_LL, FLAG_LU_BLK, FLAG_LU_DYN, FLAG_LU_GENERIC):
        out = ev.eval(torch.tensor(omega, device="cuda"), flags=FLAG_OUT_R | fl, want_P=True)
        T1, I, D = (out[k][0].cpu().numpy() for k in ("T1", "I", "Delta"))
        P = out["P"][0].cpu().numpy()
        assert (out["info"] == 0).all()
        worst = np.zeros(3)
        for f in range(0, len(omega), 4):
            eR, eI, eD = errors(ops, omega[f], T1[f], I[f], D[f], ora[0][f], ora[1][f], ora[2][f])
            worst = np.maximum(worst, [eR.max() / TOL_RI, eI.max() / TOL_RI, eD.max() / TOL_DELTA])
            po = rom.evaluate_one(float(omega[f]), out_R=True)["p"]
            for i in range(3):
                blk = P[f, i, off[i]:off[i + 1]]
                assert np.linalg.norm(blk - po[i]) <= 1e-10 * np.linalg.norm(po[i])
                assert np.all(np.delete(P[f, i], np.arange(off[i], off[i + 1])) == 0)
        assert (worst <= 1.0).all(), (fl, worst)
    w = torch.tensor([10.0, float("nan"), 1e5], device="cuda", dtype=torch.float64)
    out = ev.eval(w, flags=FLAG_OUT_R)
    assert out["info"][0].cpu().tolist() == [0, -1, 0] and torch.isnan(out["T1"][0, 1]).all()
    with pytest.raises(PodpError) as ei:
        ev.eval(w, flags=FLAG_PENCIL)
    assert ei.value.status == 4
    ev.close()


@pytest.mark.gpu
def test_N1_literal_matches_embedding_on_generated_blocks(torch_cuda):
    """Literal per-direction path vs the block embedding (both through libpodp) and vs the shared-form oracle fed
    the embedding (pinned equal to the literal formulas by test_N1_embedding_is_exact), on unequal M_i."""
    torch = torch_cuda
    from paper_2307_05590_b200 import Evaluator, FLAG_OUT_R
    from paper_2307_05590_b200 import perdir as pdir
    blk = g.make_perdir_blocks((13, 6, 9), seed=3)
    args = (blk["Kb"], blk["Cb"], blk["b0"], blk["b1"], blk["Hb"], blk["N0"], blk["S"], blk["Gx"], blk["nu"],
            blk["alpha"], blk["alpha_lb"])
    ops = pdir.embed(*args)
    omega = g.omega_grid(97)
    w = torch.tensor(omega, device="cuda")
    ev = Evaluator.per_direction(*args)
    out = ev.eval(w, flags=FLAG_OUT_R)
    T1, I, D = (out[k][0].cpu().numpy() for k in ("T1", "I", "Delta"))
    ev.close()
    from oracle.podp_oracle import certificate, mpt_I, mpt_R, solve_reduced
    for f in range(len(omega)):
        x = float(omega[f])
        P = solve_reduced(ops.K, ops.M, ops.b0, ops.b1, ops.nu, x)
        oR = oracle.to6(mpt_R(P, ops.K_R, ops.alpha))
        oI = oracle.to6(mpt_I(P, ops.M_I, ops.S, ops.H, ops.nu, ops.alpha, x))
        oD = oracle.to6(certificate(P, ops.G, ops.nu, x, ops.alpha, ops.alpha_lb)[0])
        eR, eI, eD = errors(ops, x, T1[f], I[f], D[f], oR, oI, oD)
        assert eR.max() <= TOL_RI and eI.max() <= TOL_RI and eD.max() <= TOL_DELTA, f
