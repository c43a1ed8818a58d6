"""GPU-vs-oracle parity through the C ABI (SURVEY 8(c) metric, north_star tolerances: 1e-10 per tensor entry
against the componentwise term magnitude, 1e-8 on Delta).  Marked gpu: run with `pytest -m gpu` on a B200."""
import math

import numpy as np
import pytest

import oracle
from oracle.parity import TOL_DELTA, TOL_RI, errors
from oracle.podp_oracle import solve_reduced
import podp_inputs as g

pytestmark = pytest.mark.gpu


def run_gpu(torch, ops, omega, flags=None, want_P=False, device=0):
    from paper_2307_05590_b200 import Evaluator, FLAG_OUT_R
    ev = Evaluator(ops, device=device)
    w = torch.tensor(np.asarray(omega, dtype=np.float64), device=f"cuda:{device}")
    out = ev.eval(w, flags=FLAG_OUT_R if flags is None else flags, want_P=want_P)
    torch.cuda.synchronize()
    res = {k: v.cpu().numpy() for k, v in out.items()}
    ev.close()
    return res


def check_parity(ops, omega, res, obj=0, sample=None):
    idx = range(len(omega)) if sample is None else sample
    worst = np.zeros(3)
    for f in idx:
        w = float(omega[f])
        o = oracle.evaluate_one(ops, w, out_R=True)
        eR, eI, eD = errors(ops, w, res["T1"][obj, f], res["I"][obj, f], res["Delta"][obj, f],
                            oracle.to6(o["R"]), oracle.to6(o["I"]), oracle.to6(o["Delta"]))
        worst = np.maximum(worst, [eR.max(), eI.max(), eD.max()])
    assert worst[0] <= TOL_RI, f"R parity {worst[0]:.3g}"
    assert worst[1] <= TOL_RI, f"I parity {worst[1]:.3g}"
    assert worst[2] <= TOL_DELTA, f"Delta parity {worst[2]:.3g}"
    return worst


def test_config0_full_parity_and_P(torch_cuda):
    ops, ex = g.make_config0()
    omega = g.omega_grid(200)
    res = run_gpu(torch_cuda, ops, omega, want_P=True)
    assert (res["info"] == 0).all()
    check_parity(ops, omega, res)
    for f in range(0, 200, 7):
        Po = solve_reduced(ops.K, ops.M, ops.b0, ops.b1, ops.nu, float(omega[f]))
        Pg = res["P"][0, f].T  # stored 3 x r
        assert np.linalg.norm(Pg - Po) / np.linalg.norm(Po) <= 1e-10


@pytest.mark.parametrize("r,F", [(24, 1000), (48, 333), (32, 257), (96, 61)])
def test_config_generators_parity(torch_cuda, r, F):
    ops = g.make_operators(r)
    omega = g.omega_grid(F)
    res = run_gpu(torch_cuda, ops, omega)
    assert (res["info"] == 0).all()
    check_parity(ops, omega, res)


@pytest.mark.parametrize("r", [1, 2, 7, 33, 127, 128])
def test_ragged_and_max_r(torch_cuda, r):
    rng = np.random.default_rng(r)
    if r % 2 == 0:
        ops = g.make_operators(r, seed=r)
    else:
        base = g.make_operators(r + 1, seed=r)
        # drop the last mode (still Hermitian / PSD); G keeps its structure via slot selection
        keep = np.r_[0:6, 6:6 + r, 6 + r + 1:6 + 2 * r + 1]
        ops = g.Operators(K=base.K[:r, :r], M=base.M[:r, :r], b0=base.b0[:r], b1=base.b1[:r], N0=np.eye(3),
                          S=base.S, H=base.H[:, :r], G=base.G[np.ix_(keep, keep)], nu=base.nu, alpha=base.alpha,
                          alpha_lb=base.alpha_lb)
    omega = np.sort(10 ** rng.uniform(1, 8, 37))
    res = run_gpu(torch_cuda, ops, omega)
    check_parity(ops, omega, res)


@pytest.mark.parametrize("r", [8, 24, 48, 96])
def test_generic_kernels_parity(torch_cuda, r):
    """The generic one-warp LU (PODP_FLAG_LU_GENERIC, the only kernel above padded r = 96) stays parity-green."""
    from paper_2307_05590_b200 import FLAG_OUT_R, FLAG_LU_GENERIC
    ops = g.make_config0()[0] if r == 8 else g.make_operators(r)
    omega = g.omega_grid(45)
    res = run_gpu(torch_cuda, ops, omega, flags=FLAG_OUT_R | FLAG_LU_GENERIC)
    assert (res["info"] == 0).all()
    check_parity(ops, omega, res)


def test_default_flag_outputs_Rt(torch_cuda):
    ops = g.make_operators(24)
    ops.N0 = np.array([[1.0, 0.1, 0.0], [0.1, 2.0, 0.3], [0.0, 0.3, 3.0]])
    omega = g.omega_grid(50)
    a = run_gpu(torch_cuda, ops, omega, flags=0)
    b = run_gpu(torch_cuda, ops, omega)
    n06 = oracle.to6(ops.N0)
    assert np.array_equal(a["T1"][0], n06[None, :] + b["T1"][0])
    assert np.array_equal(a["I"], b["I"]) and np.array_equal(a["Delta"], b["Delta"])


@pytest.mark.parametrize("r", [8, 48, 64, 96])
def test_no_pivot_flag_parity(torch_cuda, r):
    from paper_2307_05590_b200 import FLAG_OUT_R, FLAG_NO_PIVOT
    ops = g.make_operators(r)
    omega = g.omega_grid(97)
    res = run_gpu(torch_cuda, ops, omega, flags=FLAG_OUT_R | FLAG_NO_PIVOT)
    check_parity(ops, omega, res)


def _lu_flags(r):
    from paper_2307_05590_b200 import FLAG_LU_LL, FLAG_LU_BLK, FLAG_LU_DYN, FLAG_LU_GENERIC
    out = [("blk", FLAG_LU_BLK), ("dyn", FLAG_LU_DYN), ("generic", FLAG_LU_GENERIC)]
    if r <= 96:
        out.insert(0, ("ll", FLAG_LU_LL))
    return out


@pytest.mark.parametrize("r", [8, 16, 48, 64, 96])
def test_pivot_forcing_inputs_all_kernels(torch_cuda, r):
    """K = [[0, B], [B^H, 0]], M = diag(0, CC^H): A(omega) has an exactly zero leading r/2 x r/2 block, so every
    frequency needs row interchanges.  Every LU kernel must match the oracle (LAPACK zgesv)
    per entry, and the no-pivot variant must report the zero pivot (info = 1) -- so the suite tells a pivoted LU
    from an unpivoted one."""
    from paper_2307_05590_b200 import FLAG_OUT_R, FLAG_NO_PIVOT
    ops = g.make_pivot_forcing(r, seed=r)
    omega = g.omega_grid(67)
    for name, fl in _lu_flags(r):
        res = run_gpu(torch_cuda, ops, omega, flags=FLAG_OUT_R | fl, want_P=True)
        assert (res["info"] == 0).all(), name
        check_parity(ops, omega, res)
        for f in range(0, 67, 11):
            Po = solve_reduced(ops.K, ops.M, ops.b0, ops.b1, ops.nu, float(omega[f]))
            assert np.linalg.norm(res["P"][0, f].T - Po) / np.linalg.norm(Po) <= 1e-10, name
    res = run_gpu(torch_cuda, ops, omega, flags=FLAG_OUT_R | FLAG_NO_PIVOT)
    assert (res["info"] == 1).all() and np.isnan(res["T1"]).all()


def test_batch_objects_parity(torch_cuda):
    sig = g.batch_sigma(256)
    ops = [g.make_operators(32, seed=k, nu=g.MU0 * sig[k] * 1e-4) for k in range(5)]
    omega = g.omega_grid(129)
    res = run_gpu(torch_cuda, ops, omega)
    assert res["T1"].shape == (5, 129, 6)
    for k in range(5):
        check_parity(ops[k], omega, res, obj=k, sample=range(0, 129, 4))


def test_edge_cases_nonfinite_zero_F_singular(torch_cuda):
    torch = torch_cuda
    from paper_2307_05590_b200 import Evaluator, FLAG_OUT_R
    ops = g.make_operators(8)
    omega = np.array([10.0, np.inf, 1e5, np.nan, 0.0, 1e8])
    res = run_gpu(torch, ops, omega)
    assert list(res["info"][0]) == [0, -1, 0, -1, 0, 0]
    for f in (1, 3):
        assert np.isnan(res["T1"][0, f]).all() and np.isnan(res["I"][0, f]).all() and np.isnan(res["Delta"][0, f]).all()
    good = [0, 2, 4, 5]
    check_parity(ops, omega, res, sample=good)
    # F == 0 is a no-op
    ev = Evaluator(ops)
    out = ev.eval(torch.empty(0, dtype=torch.float64, device="cuda"))
    assert out["T1"].shape == (1, 0, 6)
    ev.close()
    # exactly singular system: K = M = 0 -> zero pivot at step 0 -> info = 1 (LAPACK getrf convention)
    z = g.Operators(**{**ops.__dict__, "K": np.zeros((8, 8), complex), "M": np.zeros((8, 8), complex)})
    res = run_gpu(torch, z, np.array([1.0, 2.0]))
    assert list(res["info"][0]) == [1, 1] and np.isnan(res["T1"]).all()


@pytest.mark.parametrize("r", [24, 32, 48, 96])
def test_edge_cases_fast_path(torch_cuda, r):
    """Non-finite omega rows and an exactly singular system on the register-resident fast path."""
    ops = g.make_operators(r)
    omega = np.array([10.0, np.nan, 3e5, -np.inf, 1e8] + list(g.omega_grid(11)))
    res = run_gpu(torch_cuda, ops, omega)
    assert list(res["info"][0][:5]) == [0, -1, 0, -1, 0]
    assert np.isnan(res["T1"][0, [1, 3]]).all() and np.isnan(res["Delta"][0, [1, 3]]).all()
    check_parity(ops, omega, res, sample=[0, 2, 4] + list(range(5, 16)))
    z = g.Operators(**{**ops.__dict__, "K": np.zeros((r, r), complex), "M": np.zeros((r, r), complex)})
    res = run_gpu(torch_cuda, z, np.array([1.0, 2.0, 3.0]))
    assert list(res["info"][0]) == [1, 1, 1] and np.isnan(res["I"]).all()
    # singular at a later step: K = diag(1..r) with a zero at position 5, M = 0 -> zero pivot at step 5
    d = np.arange(1.0, r + 1)
    d[5] = 0.0
    z = g.Operators(**{**ops.__dict__, "K": np.diag(d).astype(complex), "M": np.zeros((r, r), complex)})
    res = run_gpu(torch_cuda, z, np.array([1.0, 2.0]))
    assert list(res["info"][0]) == [6, 6]


@pytest.mark.parametrize("r", [8, 24, 40, 48, 56, 64, 72, 80, 96])
def test_all_lu_kernels_parity_and_singular(torch_cuda, r):
    """Every LU kernel (left-looking one-warp 'll' for padded r <= 64, lock-step blocked 'blk', dynamically scheduled
    'dyn', generic) stays parity-green on every size class, including a non-finite omega and a zero pivot at a
    later panel (LAPACK info = k+1)."""
    from paper_2307_05590_b200 import FLAG_OUT_R
    ops = g.make_operators(r, seed=r + 1)
    omega = np.r_[g.omega_grid(61), [np.inf]]
    d = np.arange(1.0, r + 1)
    k0 = min(r - 1, 13)
    d[k0] = 0.0
    z = g.Operators(**{**ops.__dict__, "K": np.diag(d).astype(complex), "M": np.zeros((r, r), complex)})
    for name, fl in _lu_flags(r):
        res = run_gpu(torch_cuda, ops, omega, flags=FLAG_OUT_R | fl)
        assert (res["info"][0][:61] == 0).all() and res["info"][0][61] == -1, name
        check_parity(ops, omega, res, sample=range(61))
        res = run_gpu(torch_cuda, z, np.array([1.0, 2.0]), flags=FLAG_OUT_R | fl)
        assert list(res["info"][0]) == [k0 + 1, k0 + 1] and np.isnan(res["T1"]).all(), name


def test_lu_kernel_selection_errors(torch_cuda):
    from paper_2307_05590_b200 import Evaluator, PodpError, FLAG_LU_LL, FLAG_LU_BLK, FLAG_NO_PIVOT
    torch = torch_cuda
    ev = Evaluator(g.make_operators(104))
    w = torch.tensor(g.omega_grid(5), device="cuda")
    with pytest.raises(PodpError) as ei:
        ev.eval(w, flags=FLAG_LU_LL)            # not instantiated above padded r = 96
    assert ei.value.status == 4
    with pytest.raises(PodpError) as ei:
        ev.eval(w, flags=FLAG_LU_LL | FLAG_LU_BLK)
    assert ei.value.status == 1
    with pytest.raises(PodpError) as ei:
        ev.eval(w, flags=FLAG_LU_BLK | FLAG_NO_PIVOT)
    assert ei.value.status == 4
    ev.close()


def test_invariants_scaling_bitwise(torch_cuda):
    """Remark 6.2, pin C8 on the GPU path: power-of-two scaling is exact -> bitwise."""
    o = g.make_operators(24)
    Dg = np.ones(6 + 2 * o.r)
    Dg[[1, 3, 5]] = 4.0
    o2 = g.Operators(**{**o.__dict__, "alpha": 2 * o.alpha, "nu": 4 * o.nu, "b1": 4 * o.b1, "S": 4 * o.S,
                        "H": 4 * o.H, "G": (Dg[:, None] * o.G) * Dg[None, :]})
    omega = g.omega_grid(64)
    a = run_gpu(torch_cuda, o2, omega)
    b = run_gpu(torch_cuda, o, 4 * omega)
    for k in ("T1", "I", "Delta"):
        assert np.array_equal(a[k], 8 * b[k]), k


def test_symmetry_and_sign_structure_config0(torch_cuda):
    ops, _ = g.make_config0()
    omega = g.omega_grid(200)
    res = run_gpu(torch_cuda, ops, omega)
    for f in range(200):
        R = oracle.from6(res["T1"][0, f])
        I = oracle.from6(res["I"][0, f])
        assert np.max(np.linalg.eigvalsh(R)) <= 1e-12 * np.abs(R).max()
        assert np.min(np.linalg.eigvalsh(I)) >= -1e-12 * np.abs(I).max()
        assert (res["Delta"][0, f] >= 0).all()


def test_select_matches_oracle_on_gpu_delta(torch_cuda):
    torch = torch_cuda
    from paper_2307_05590_b200 import Evaluator
    ops = g.make_operators(24)
    omega = g.omega_grid(20000)
    snap = g.snapshot_grid(13)
    ev = Evaluator(ops)
    w = torch.tensor(omega, device="cuda")
    out = ev.eval(w)
    D = out["Delta"][0]
    wn, idx, Lam, lam_n = ev.select(w, D, snap, n_star=2)
    Dh = D.cpu().numpy()
    ow, oidx, oLam, olam = oracle.select(omega, Dh, snap, 2)
    assert list(idx) == oidx and list(wn) == ow and Lam == oLam
    assert [x if x is not None else -1.0 for x in olam] == list(lam_n)
    for theta in (1.0, 0.5, 1e-3):
        wn, idx, Lam, _ = ev.select(w, D, snap, n_star=12, theta=theta)
        ow, oidx, oLam, _ = oracle.select(omega, Dh, snap, 12, theta=theta)
        assert list(idx) == oidx and Lam == oLam
    # too many requested intervals -> PODP_ERR_NO_CANDIDATES
    from paper_2307_05590_b200 import PodpError
    with pytest.raises(PodpError) as ei:
        ev.select(w, D, snap, n_star=13)
    assert ei.value.status == 7
    ev.close()


def test_select_ties_and_nan(torch_cuda):
    torch = torch_cuda
    from paper_2307_05590_b200 import Evaluator
    ev = Evaluator(g.make_operators(8))
    omega = np.linspace(1.0, 5.0, 4001)
    snap = np.array([1.0, 2.0, 3.0, 4.0, 5.0])
    D = np.zeros((4001, 6))
    D[1500:1510, 2] = 7.0       # ties inside interval [2,3) -> lowest index 1500
    D[2600, 0] = 7.0            # tie across intervals -> lower interval index wins for N*=1
    D[100, 3] = np.nan
    D[3000, :] = -0.0
    wd, Dd = torch.tensor(omega, device="cuda"), torch.tensor(D, device="cuda")
    wn, idx, Lam, lam_n = ev.select(wd, Dd, snap, n_star=1)
    ow, oidx, oLam, _ = oracle.select(omega, D, snap, 1)
    assert list(idx) == oidx == [1500] and Lam == oLam == 7.0
    wn, idx, Lam, lam_n = ev.select(wd, Dd, snap, n_star=2)
    assert list(idx) == oracle.select(omega, D, snap, 2)[1] == [1500, 2600]
    ev.close()


def test_eval_host_matches_device(torch_cuda):
    from paper_2307_05590_b200 import Evaluator, FLAG_OUT_R
    ops = g.make_operators(48)
    omega = g.omega_grid(1001)
    ev = Evaluator(ops)
    h = ev.eval_host(omega, flags=FLAG_OUT_R)
    d = run_gpu(torch_cuda, ops, omega)
    for k in ("T1", "I", "Delta", "info"):
        assert np.array_equal(h[k], d[k]), k
    ev.close()


def test_eval_host_batch_nan(torch_cuda):
    """Host entry with several objects and a failed frequency: results must equal the device entry bit for bit."""
    torch = torch_cuda
    from paper_2307_05590_b200 import Evaluator, FLAG_OUT_R
    ops = [g.make_operators(24, seed=k) for k in range(2)]
    omega = g.omega_grid(90_001)
    omega[777] = np.nan                       # a failed frequency inside a chunk
    ev = Evaluator(ops)
    h = ev.eval_host(omega, flags=FLAG_OUT_R)
    d = ev.eval(torch.tensor(omega, device="cuda"), flags=FLAG_OUT_R)
    torch.cuda.synchronize()
    for k in ("T1", "I", "Delta"):
        assert np.array_equal(h[k], d[k].cpu().numpy(), equal_nan=True), k
    assert np.array_equal(h["info"], d["info"].cpu().numpy())
    assert (h["info"][:, 777] == -1).all() and (np.delete(h["info"], 777, axis=1) == 0).all()
    ev.close()


@pytest.mark.parametrize("r,F", [(8, 8192), (24, 20_001), (48, 9_999)])
def test_eval_host_overlapped_copy(torch_cuda, r, F):
    """One object and F >= 8192: podp_eval_host runs the contraction as two launches and copies the first half of the
    outputs back while the second half is computed.  Results (with failed frequencies in both halves and at the
    split) must equal the device entry bit for bit, and a second call on the same context must too."""
    torch = torch_cuda
    from paper_2307_05590_b200 import Evaluator, FLAG_OUT_R
    ops = g.make_operators(r)
    omega = g.omega_grid(F)
    F1 = (F // 2) // 64 * 64
    for k in (5, F1 - 1, F1, F - 2):
        omega[k] = np.nan
    ev = Evaluator(ops)
    d = ev.eval(torch.tensor(omega, device="cuda"), flags=FLAG_OUT_R)
    torch.cuda.synchronize()
    for _ in range(2):
        h = ev.eval_host(omega, flags=FLAG_OUT_R)
        for k in ("T1", "I", "Delta"):
            assert np.array_equal(h[k], d[k].cpu().numpy(), equal_nan=True), k
        assert np.array_equal(h["info"], d["info"].cpu().numpy())
    assert (h["info"][0, [5, F1 - 1, F1, F - 2]] == -1).all() and np.isnan(h["T1"][0, F1]).all()
    ev.close()


@pytest.mark.slow
@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
def test_full_size_configs_sampled(torch_cuda, cfg):
    """BASELINE configs at full size in the bench launch configuration; parity on a sample of outputs the
    oracle computes one by one (plus properties that hold at any size)."""
    torch = torch_cuda
    from paper_2307_05590_b200 import Evaluator, FLAG_OUT_R
    c = g.make_config(cfg)
    omega = c["omega"]
    ev = Evaluator(c["ops"])
    w = torch.tensor(omega, device="cuda")
    out = ev.eval(w, flags=FLAG_OUT_R, info=True)
    torch.cuda.synchronize()
    F = len(omega)
    rng = np.random.default_rng(cfg)
    sample = sorted(set([0, F - 1, F // 2] + list(rng.integers(0, F, 40))))
    n_obj = len(c["ops"])
    objs = [0, n_obj - 1, n_obj // 2] if n_obj > 1 else [0]
    for k in objs:
        res = {key: out[key][k][sample].cpu().numpy()[None] for key in ("T1", "I", "Delta")}
        check_parity(c["ops"][k], omega[sample], res)
    assert int(out["info"].abs().sum()) == 0
    assert torch.isfinite(out["Delta"]).all() and (out["Delta"] >= 0).all()
    if cfg == 4:
        wn, idx, Lam, lam_n = ev.select(w, out["Delta"][0], c["snap"], n_star=2)
        ow, oidx, oLam, _ = oracle.select(omega, out["Delta"][0].cpu().numpy(), c["snap"], 2)
        assert list(idx) == oidx and Lam == oLam
    ev.close()


@pytest.mark.parametrize("r,F", [(8, 200), (24, 500), (48, 333), (96, 61), (32, 129)])
def test_pencil_solver_parity(torch_cuda, r, F):
    """NEXT row N3: the pencil reformulation (P = Z (I + i omega nu Lambda)^{-1} Z^H B) matches the LU oracle."""
    from paper_2307_05590_b200 import FLAG_OUT_R, FLAG_PENCIL
    ops = g.make_config0()[0] if r == 8 else g.make_operators(r)
    omega = g.omega_grid(F)
    res = run_gpu(torch_cuda, ops, omega, flags=FLAG_OUT_R | FLAG_PENCIL, want_P=True)
    assert (res["info"] == 0).all()
    check_parity(ops, omega, res)
    for f in range(0, F, max(1, F // 13)):
        Po = solve_reduced(ops.K, ops.M, ops.b0, ops.b1, ops.nu, float(omega[f]))
        assert np.linalg.norm(res["P"][0, f].T - Po) / np.linalg.norm(Po) <= 1e-10
    # without the debug P output the MPT/certificate kernel runs in pencil coordinates (y, Z^H X Z; diagonal
    # K_R and M_I forms since K_R = K and M_I = M here)
    res_y = run_gpu(torch_cuda, ops, omega, flags=FLAG_OUT_R | FLAG_PENCIL)
    assert (res_y["info"] == 0).all()
    check_parity(ops, omega, res_y)


def test_pencil_batch_and_unsupported(torch_cuda):
    torch = torch_cuda
    from paper_2307_05590_b200 import Evaluator, FLAG_OUT_R, FLAG_PENCIL, PodpError
    sig = g.batch_sigma(256)
    ops = [g.make_operators(32, seed=k, nu=g.MU0 * sig[k] * 1e-4) for k in range(4)]
    omega = g.omega_grid(77)
    res = run_gpu(torch, ops, omega, flags=FLAG_OUT_R | FLAG_PENCIL)
    for k in range(4):
        check_parity(ops[k], omega, res, obj=k, sample=range(0, 77, 5))
    # K not positive definite -> the pencil path is refused (the LU path still works)
    o = g.make_operators(8)
    o = g.Operators(**{**o.__dict__, "K": o.K - 20.0 * np.eye(8)})
    ev = Evaluator(o)
    with pytest.raises(PodpError) as ei:
        ev.eval(torch.tensor(omega, device="cuda"), flags=FLAG_PENCIL)
    assert ei.value.status == 4
    ev.close()


@pytest.mark.parametrize("r", [8, 48, 96])
def test_pencil_illconditioned_K(torch_cuda, r):
    """N3 on ill-conditioned K (its Z = L^{-H} V has condition number sqrt(kappa(K))).

    kappa = 1e4: the standard gate against the FP64 oracle.  kappa = 1e8: there the FP64 oracle itself is only
    accurate to ~kappa u (1-2e-9 against an 80-bit LU, measured), and two FP64 methods that do not share rounding
    (LAPACK LU vs Cholesky + eigen pencil) differ by that much; SURVEY 8(c)'s adjudication rule applies: each GPU
    path's worst error over the sweep against the 80-bit re-evaluation (oracle/extended.py) must be <= 4x the FP64
    oracle's worst error over the sweep (or <= the north_star tolerance).  (The LU kernel differs from LAPACK's LU
    by ~2e-9 there too: a different pivot key and operation order, measured.)"""
    from oracle.extended import evaluate_one_ld
    from paper_2307_05590_b200 import FLAG_OUT_R, FLAG_PENCIL
    ops = g.make_illconditioned(r, 1e4, seed=r)
    omega = g.omega_grid(53)
    for fl in (FLAG_OUT_R | FLAG_PENCIL, FLAG_OUT_R):
        res = run_gpu(torch_cuda, ops, omega, flags=fl)
        assert (res["info"] == 0).all()
        check_parity(ops, omega, res)
    ops = g.make_illconditioned(r, 1e8, seed=r)
    omega = g.omega_grid(29)
    res_lu = run_gpu(torch_cuda, ops, omega, flags=FLAG_OUT_R)
    assert (res_lu["info"] == 0).all()
    res_pe = run_gpu(torch_cuda, ops, omega, flags=FLAG_OUT_R | FLAG_PENCIL)
    assert (res_pe["info"] == 0).all()
    worst_o = np.zeros(3)
    worst_g = {"lu": np.zeros(3), "pencil": np.zeros(3)}
    for f, w in enumerate(omega):
        w = float(w)
        t = evaluate_one_ld(ops, w)
        o = oracle.evaluate_one(ops, w, out_R=True)
        eo = errors(ops, w, oracle.to6(o["R"]), oracle.to6(o["I"]), oracle.to6(o["Delta"]), t["R6"], t["I6"], t["D6"])
        worst_o = np.maximum(worst_o, [x.max() for x in eo])
        for name, res in (("lu", res_lu), ("pencil", res_pe)):
            eg = errors(ops, w, res["T1"][0, f], res["I"][0, f], res["Delta"][0, f], t["R6"], t["I6"], t["D6"])
            worst_g[name] = np.maximum(worst_g[name], [x.max() for x in eg])
    # worst over the sweep against the FP64 oracle's worst over the sweep (per omega the oracle can be lucky)
    bound = np.maximum([TOL_RI, TOL_RI, TOL_DELTA], 4.0 * worst_o)
    for name, wg in worst_g.items():
        assert np.all(wg <= bound), (name, wg, worst_o)
    worst_ratio = max(float(np.max(wg / np.maximum(worst_o, 1e-300))) for wg in worst_g.values())
    print(f"r={r} kappa=1e8: worst GPU/oracle error ratio against 80-bit {worst_ratio:.3g}")


def test_N4_invariants_and_voltage_parity(torch_cuda):
    torch = torch_cuda
    import paper_2307_05590_b200 as pb
    ops = g.make_operators(24)
    omega = g.omega_grid(301)
    ev = pb.Evaluator(ops)
    out = ev.eval(torch.tensor(omega, device="cuda"))
    eR, eI = pb.invariants(out["T1"], out["I"])
    T1, I = out["T1"][0].cpu().numpy(), out["I"][0].cpu().numpy()
    oR, oI = oracle.invariants((T1, I))
    for gpu, ora in ((eR[0].cpu().numpy(), oR), (eI[0].cpu().numpy(), oI)):
        scale = np.abs(ora).max(axis=1, keepdims=True)
        assert np.max(np.abs(gpu - ora) / scale) <= 1e-13
    rng = np.random.default_rng(0)
    hx, hm = rng.standard_normal((5, 3)), rng.standard_normal((5, 3))
    V = pb.coil_voltage(out["T1"], out["I"], hx, hm)[0].cpu().numpy()
    Vo = oracle.coil_voltage(T1, I, hx, hm)
    assert np.max(np.abs(V - Vo) / np.abs(Vo).max()) <= 1e-14
    # Remark 6.2 relabelling helper is exact
    om2, sc = pb.scale_signature(omega, {"T1": out["T1"], "I": out["I"], "Delta": out["Delta"]}, 2.0)
    assert np.array_equal(om2, omega / 4.0) and torch.equal(sc["I"], 8.0 * out["I"])
    ev.close()


@pytest.mark.parametrize("r", [8, 48, 56, 96])
def test_lu_kernels_deterministic_across_launch_shapes(torch_cuda, r):
    """Race evidence without compute-sanitizer (closed on this pool): every LU kernel computes one frequency's result
    with a fixed operation order, independent of which warp/CTA/SM runs it and of what runs beside it.  So repeated
    full-GPU launches, and the same frequencies evaluated alone or shifted to other warps, must agree BIT FOR BIT; a
    shared-memory race, a missing barrier or a scheduling-dependent task order shows up as a difference."""
    torch = torch_cuda
    from paper_2307_05590_b200 import Evaluator, FLAG_OUT_R
    ops = g.make_operators(r) if r != 8 else g.make_config0()[0]
    omega = g.omega_grid(4001)
    w = torch.tensor(omega, device="cuda")
    ev = Evaluator(ops)
    for name, fl in _lu_flags(r):
        ref = None
        for rep in range(3):
            out = ev.eval(w, flags=FLAG_OUT_R | fl)
            cur = torch.cat([out["T1"][0], out["I"][0], out["Delta"][0]], dim=1).cpu().numpy()
            if ref is None:
                ref = cur
            else:
                assert np.array_equal(ref.view(np.uint64), cur.view(np.uint64)), (name, rep)
        for sl in (slice(0, 1), slice(1, 34), slice(2000, 2077), slice(3999, 4001)):
            out = ev.eval(w[sl].contiguous(), flags=FLAG_OUT_R | fl)
            cur = torch.cat([out["T1"][0], out["I"][0], out["Delta"][0]], dim=1).cpu().numpy()
            assert np.array_equal(ref[sl].view(np.uint64), cur.view(np.uint64)), (name, sl)
    ev.close()


@pytest.mark.parametrize("sigma", [1e-160, 1e155])
def test_tiny_and_huge_pivots(torch_cuda, sigma):
    """Pivots whose |p|^2 leaves the normal double range (|p| ~ 1e-160 or 1e155): every LU kernel takes its
    call-free scaled reciprocal there (the fast reciprocal alone would return NaN rows with info = 0).
    K, M and b0, b1 scaled by sigma (K_R = the unscaled K) leave P, R and Delta unchanged in exact arithmetic, so they
    are gated against the oracle on the UNSCALED problem (I is not: its nu p^H M p term scales with sigma)."""
    from paper_2307_05590_b200 import FLAG_OUT_R
    for r in (8, 48, 96):
        o = g.make_operators(r)
        ops = g.Operators(**{**o.__dict__, "K": o.K * sigma, "M": o.M * sigma, "K_R": o.K.copy(),
                             "b0": o.b0 * sigma, "b1": o.b1 * sigma})
        omega = g.omega_grid(41)
        for name, fl in _lu_flags(r):
            res = run_gpu(torch_cuda, ops, omega, flags=FLAG_OUT_R | fl, want_P=True)
            assert (res["info"] == 0).all(), (r, name)
            for f, w in enumerate(omega):
                w = float(w)
                ora = oracle.evaluate_one(o, w, out_R=True)
                assert np.linalg.norm(res["P"][0, f].T - ora["P"]) <= 1e-10 * np.linalg.norm(ora["P"]), (r, name)
                eR, _eI, eD = errors(o, w, res["T1"][0, f], oracle.to6(ora["I"]), res["Delta"][0, f],
                                     oracle.to6(ora["R"]), oracle.to6(ora["I"]), oracle.to6(ora["Delta"]))
                assert eR.max() <= TOL_RI and eD.max() <= TOL_DELTA, (r, name, w)


def test_release_workspace_and_reuse(torch_cuda):
    """podp_release_workspace trims the library's pool; evaluations before and after agree bit for bit."""
    torch = torch_cuda
    import paper_2307_05590_b200 as pb
    ops = g.make_operators(24)
    w = torch.tensor(g.omega_grid(3001), device="cuda")
    ev = pb.Evaluator(ops)
    a = ev.eval(w, flags=pb.FLAG_OUT_R)
    torch.cuda.synchronize()
    pb.release_workspace(0)
    b = ev.eval(w, flags=pb.FLAG_OUT_R)
    torch.cuda.synchronize()
    for k in ("T1", "I", "Delta"):
        assert torch.equal(a[k], b[k])
    ev.close()
    with pytest.raises(pb.PodpError):
        pb.release_workspace(7)


@pytest.mark.parametrize("r", [8, 24, 40, 48, 56, 64, 96])
def test_batch_objects_every_lu_path(torch_cuda, r):
    """Multi-object launches through every left-looking variant (K/M in shared memory walked object by object at
    r <= 40, the tensor-memory variant at 48 <= r <= 64, the L2-gather variant at r = 96): per-object parity against
    the oracle, including a zero-pivot object and a non-finite omega, and bit-identical results for the same object
    evaluated alone (the object walk must not leak one object's K and M into another's solves)."""
    torch = torch_cuda
    from paper_2307_05590_b200 import Evaluator, FLAG_OUT_R
    sig = g.batch_sigma(256)
    ops = [g.make_operators(r, seed=k, nu=g.MU0 * sig[k] * 1e-4) for k in range(4)]
    ops[2] = g.make_pivot_forcing(r, seed=5) if r % 2 == 0 else ops[2]
    omega = g.omega_grid(211)
    omega[17] = float("nan")
    res = run_gpu(torch, ops, omega)
    ok = [f for f in range(211) if f != 17]
    for k in range(4):
        assert res["info"][k, 17] == -1 and np.isnan(res["T1"][k, 17]).all()
        assert (res["info"][k, ok] == 0).all()
        check_parity(ops[k], omega, res, obj=k, sample=[f for f in range(0, 211, 9) if f != 17])
    for k in (0, 2):
        alone = run_gpu(torch, [ops[k]], omega)
        for q in ("T1", "I", "Delta"):
            assert np.array_equal(np.nan_to_num(alone[q][0]).view(np.uint64), np.nan_to_num(res[q][k]).view(np.uint64)), (k, q)


@pytest.mark.parametrize("r,F", [(24, 333), (48, 257), (96, 61), (20, 49)])
def test_mpt_gemm_variant_parity(torch_cuda, r, F):
    """A/B variant of the contraction (PODP_FLAG_MPT_GEMM: DMMA GEMMs over the solution panel, bulk-copy staging):
    per-entry parity against the oracle, including a ragged last tile; unsupported cases are refused."""
    torch = torch_cuda
    from paper_2307_05590_b200 import Evaluator, FLAG_MPT_GEMM, FLAG_OUT_R, PodpError
    ops = g.make_operators(r)
    omega = g.omega_grid(F)
    if (r + 7) // 8 * 8 not in (24, 48, 96):
        ev = Evaluator(ops)
        with pytest.raises(PodpError) as ei:
            ev.eval(torch.tensor(omega, device="cuda"), flags=FLAG_MPT_GEMM)
        assert ei.value.status == 4
        ev.close()
        return
    res = run_gpu(torch, ops, omega, flags=FLAG_OUT_R | FLAG_MPT_GEMM)
    assert (res["info"] == 0).all()
    check_parity(ops, omega, res)


@pytest.mark.parametrize("r,F", [(48, 257), (48, 5), (47, 131), (41, 64)])
def test_mpt_paired_and_single_kernels_parity(torch_cuda, r, F):
    """The default contraction kernel and the A/B kernel with two frequencies per lane (PODP_FLAG_MPT_PAIR, padded
    r = 48) both match the oracle per entry, including ragged last tiles (F not a multiple of 32, odd F: the second
    frequency of a lane pair is missing) and padded r."""
    torch = torch_cuda
    from paper_2307_05590_b200 import FLAG_MPT_PAIR, FLAG_OUT_R
    ops = g.make_operators(r if r % 2 == 0 else r + 1)
    if r % 2:
        keep = np.r_[0:6, 6:6 + r, 6 + r + 1:6 + r + 1 + r]
        ops = g.Operators(K=ops.K[:r, :r], M=ops.M[:r, :r], b0=ops.b0[:r], b1=ops.b1[:r], N0=ops.N0, S=ops.S,
                          H=ops.H[:, :r], G=ops.G[np.ix_(keep, keep)], nu=ops.nu, alpha=ops.alpha,
                          alpha_lb=ops.alpha_lb)
    omega = g.omega_grid(F)
    for flags in (FLAG_OUT_R, FLAG_OUT_R | FLAG_MPT_PAIR):
        res = run_gpu(torch, ops, omega, flags=flags)
        assert (res["info"] == 0).all()
        check_parity(ops, omega, res)
