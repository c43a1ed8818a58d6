"""Oracle pins: the CPU oracle checked against what the paper and mathematics fix,
independently of its own formulas.  CPU only (-m "not gpu")."""
import json
import math
import os

import numpy as np
import pytest
import scipy.linalg

import oracle
from oracle import fullorder
from oracle.podp_oracle import certificate, mpt_I, mpt_R, residual_coeffs, solve_reduced
import podp_inputs as g

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
U = np.finfo(float).eps / 2


@pytest.fixture(scope="module")
def c0():
    return g.make_config0()


@pytest.fixture(scope="module")
def c1ops():
    return g.make_operators(24)


def test_constants_golden():
    gd = json.load(open(os.path.join(GOLDEN, "constants.json")))
    assert g.MU0 == gd["mu0"]
    assert abs(g.NU_DEFAULT - gd["nu_config0"]) <= 2 * U * gd["nu_config0"]
    assert abs(gd["mu0"] * gd["sigma_config0"] * gd["alpha_config0"] ** 2 - gd["nu_config0"]) < 1e-18


# ---------------------------------------------------------------- C1: solver backward error (a3)
@pytest.mark.parametrize("omega", [10.0, 3.3e3, 1e6, 1e8])
def test_C1_backward_error(c1ops, omega):
    o = c1ops
    P = solve_reduced(o.K, o.M, o.b0, o.b1, o.nu, omega)
    A = o.K + 1j * omega * o.nu * o.M
    B = o.b0 + omega * o.b1
    be = np.linalg.norm(A @ P - B) / (np.linalg.norm(A) * np.linalg.norm(P))
    assert be <= 10 * o.r * U


# ---------------------------------------------------------------- C2: closed forms (a2-a3)
def test_C2_scalar_r1():
    rng = np.random.default_rng(5)
    k, m = 2.5, 0.75
    b0 = rng.standard_normal((1, 3)) + 1j * rng.standard_normal((1, 3))
    b1 = rng.standard_normal((1, 3)) + 1j * rng.standard_normal((1, 3))
    nu = g.NU_DEFAULT
    for w in [10.0, 1e4, 1e8]:
        P = solve_reduced(np.array([[k]]), np.array([[m]]), b0, b1, nu, w)
        # scalar division ("M=1 -> scalar division")
        expect = (b0[0] + w * b1[0]) / complex(k, w * nu * m)
        assert np.allclose(P[0], expect, rtol=4 * U, atol=0)


def test_C2_diagonal_componentwise():
    rng = np.random.default_rng(6)
    r = 7
    kd = 1 + rng.random(r)
    md = rng.random(r)
    b0 = rng.standard_normal((r, 3)) + 1j * rng.standard_normal((r, 3))
    b1 = rng.standard_normal((r, 3)) + 1j * rng.standard_normal((r, 3))
    w = 5e5
    P = solve_reduced(np.diag(kd).astype(complex), np.diag(md).astype(complex), b0, b1, g.NU_DEFAULT, w)
    expect = (b0 + w * b1) / (kd + 1j * w * g.NU_DEFAULT * md)[:, None]
    assert np.allclose(P, expect, rtol=8 * U, atol=0)


# ---------------------------------------------------------------- C3: Galerkin reproduction (a3, a5)
def test_C3_galerkin_reproduction(c0):
    ops, ex = c0
    ops2, ex2, y = g.make_galerkin_variant(ops, ex)
    for w in [10.0, 1e3, 1e5, 1e8]:
        P = solve_reduced(ops2.K, ops2.M, ops2.b0, ops2.b1, ops2.nu, w)
        assert np.max(np.abs(P - y)) / np.max(np.abs(y)) < 1e-13
        D, n, X = certificate(P, ops2.G, ops2.nu, w, ops2.alpha, ops2.alpha_lb)
        # true residual is exactly 0: Gram-Delta is rounding only, tiny relative to its term magnitude
        Wt = residual_coeffs(P, ops2.nu, w)
        term = np.abs(Wt).T @ np.abs(ops2.G) @ np.abs(Wt)
        assert np.all(n <= 1e-13 * np.diag(term))
        # and the explicit full-order residual vanishes too
        res = fullorder.full_residual(ex2.K_full, ex2.M_full, ex2.B0f, ex2.B1f, ex2.U, P, ops2.nu, w)
        scale = np.linalg.norm(ex2.B0f + w * ex2.B1f, axis=0)
        assert np.all(np.linalg.norm(res, axis=0) <= 1e-12 * scale)


# ---------------------------------------------------------------- C4: reduced vs full-order reconstruction (a4)
@pytest.mark.parametrize("omega", [10.0, 1.7e2, 4e4, 1e6, 1e8])
def test_C4_mm_equals_fmm_on_reconstruction(c0, omega):
    ops, ex = c0
    out = oracle.evaluate_one(ops, omega, out_R=True)
    Q = fullorder.reconstruct(ex.U, out["P"])
    Rf = fullorder.fmm_R(Q, ex.K_full, ops.alpha)
    If = fullorder.fmm_I(Q, ex.v, ex.C_full, ops.alpha, omega)
    assert np.max(np.abs(out["R"] - Rf)) <= 1e-11 * np.max(np.abs(Rf))
    assert np.max(np.abs(out["I"] - If)) <= 1e-11 * np.max(np.abs(If))
    # and Rt = N0 + R
    outt = oracle.evaluate_one(ops, omega)
    assert np.array_equal(outt["T1"], np.eye(3) + out["R"])


# ---------------------------------------------------------------- C5: U = I exact (a4)
def test_C5_identity_basis_equals_full_order():
    rng = np.random.default_rng(11)
    N = 8
    A = rng.standard_normal((N, N)) + 1j * rng.standard_normal((N, N))
    K_full = A.conj().T @ A + 0.5 * np.eye(N)
    C = rng.standard_normal((4, N)) + 1j * rng.standard_normal((4, N))
    M_full = C.conj().T @ C
    Ub = np.eye(N)
    b0 = rng.standard_normal((N, 3)) + 1j * rng.standard_normal((N, 3))
    b1 = rng.standard_normal((N, 3)) + 1j * rng.standard_normal((N, 3))
    v = rng.standard_normal((N, 3))
    nu, alpha = g.NU_DEFAULT, 1e-2
    C_full = nu * M_full
    S = np.real(v.T @ C_full @ v)
    H = v.T @ C_full @ Ub
    K = Ub.conj().T @ K_full @ Ub
    M = Ub.conj().T @ M_full @ Ub
    assert np.array_equal(K, K_full) and np.array_equal(M, M_full)
    ops = g.Operators(K=K, M=M, b0=b0, b1=b1, N0=np.eye(3), S=0.5 * (S + S.T), H=H,
                      G=np.eye(6 + 2 * N, dtype=complex), nu=nu, alpha=alpha, alpha_lb=1.0)
    for w in [10.0, 1e5, 1e8]:
        out = oracle.evaluate_one(ops, w, out_R=True)
        q = fullorder.full_solve(K_full, M_full, b0, b1, nu, w)
        assert np.max(np.abs(out["P"] - q)) <= 1e-14 * np.max(np.abs(q))
        Rf = fullorder.fmm_R(q, K_full, alpha)
        If = fullorder.fmm_I(q, v, C_full, alpha, w)
        assert np.max(np.abs(out["R"] - Rf)) <= 1e-13 * np.max(np.abs(Rf))
        # I's summands cancel at high omega: compare against the term magnitude (|q|+|v|)^T |C| (|q|+|v|)
        a = np.abs(q) + np.abs(v)
        termI = w * alpha ** 3 / 4 * np.max(a.T @ np.abs(C_full) @ a)
        assert np.max(np.abs(out["I"] - If)) <= 1e-14 * termI


# ---------------------------------------------------------------- C6: symmetry / definiteness (a4)
def test_C6_symmetry_and_definiteness(c0):
    ops, _ = c0
    for w in g.omega_grid(23):
        out = oracle.evaluate_one(ops, w, out_R=True)
        R, I, D = out["R"], out["I"], out["Delta"]
        assert np.array_equal(R, R.T) and np.array_equal(I, I.T) and np.array_equal(D, D.T)
        # R is minus a Gram (K_R >= 0) -> R <= 0 ; I is a nu-weighted Gram (Gram-consistent S, H) -> I >= 0
        assert np.max(np.linalg.eigvalsh(R)) <= 1e-12 * np.max(np.abs(R))
        assert np.min(np.linalg.eigvalsh(I)) >= -1e-12 * np.max(np.abs(I))


# ---------------------------------------------------------------- C7: limits (a4)
def test_C7_low_frequency_limits(c1ops):
    o = c1ops
    # R(omega -> 0) -> -(alpha^3/4) Re(b0^H K^{-1} b0) (one Cholesky solve, a different LAPACK path)
    cf = scipy.linalg.cho_factor(o.K)
    lim = np.zeros((3, 3))
    for i in range(3):
        for j in range(3):
            lim[i, j] = -(o.alpha ** 3 / 4) * np.real(np.vdot(o.b0[:, i], scipy.linalg.cho_solve(cf, o.b0[:, j])))
    out = oracle.evaluate_one(o, 1e-9, out_R=True)
    assert np.max(np.abs(out["R"] - lim)) <= 1e-6 * np.max(np.abs(lim))
    out0 = oracle.evaluate_one(o, 0.0, out_R=True)
    assert np.max(np.abs(out0["R"] - lim)) <= 1e-12 * np.max(np.abs(lim))
    # I -> 0 linearly as omega -> 0 (omega prefactor)
    i1 = oracle.evaluate_one(o, 1e-6)["I"]
    i2 = oracle.evaluate_one(o, 2e-6)["I"]
    assert np.max(np.abs(i1)) < 1e-12
    assert np.allclose(i2, 2 * i1, rtol=1e-6, atol=0)
    assert np.array_equal(out0["I"], np.zeros((3, 3)))


def test_C7_zero_solution(c1ops):
    o = g.Operators(**{**c1ops.__dict__, "b0": np.zeros_like(c1ops.b0), "b1": np.zeros_like(c1ops.b1)})
    for w in [10.0, 1e7]:
        out = oracle.evaluate_one(o, w, out_R=True)
        assert np.array_equal(out["R"], np.zeros((3, 3)))
        assert np.array_equal(out["I"], (w * o.alpha ** 3 / 4) * o.S)


# ---------------------------------------------------------------- C8: Remark 6.2 scaling (a2-a5), bitwise
def test_C8_size_scaling_bitwise(c1ops):
    o = c1ops
    Dg = np.ones(6 + 2 * o.r)
    Dg[[1, 3, 5]] = 4.0
    o2 = g.Operators(**{**o.__dict__, "alpha": 2 * o.alpha, "nu": 4 * o.nu, "b1": 4 * o.b1, "S": 4 * o.S,
                        "H": 4 * o.H, "G": (Dg[:, None] * o.G) * Dg[None, :]})
    for w in [10.0, 2.5e3, 1e6, 2.5e7]:
        a = oracle.evaluate_one(o2, w, out_R=True)
        b = oracle.evaluate_one(o, 4 * w, out_R=True)
        assert np.array_equal(a["P"], b["P"])
        for key in ("R", "I", "Delta"):
            assert np.array_equal(a[key], 8 * b[key]), key


# ---------------------------------------------------------------- C9: conjugation invariance (U1)
def test_C9_conjugation_invariance(c1ops):
    o = c1ops
    oc = g.Operators(**{**o.__dict__, "K": o.K.conj(), "M": o.M.conj(), "b0": o.b0.conj(), "b1": o.b1.conj(),
                        "H": o.H.conj(), "G": o.G.conj()})
    for w in [10.0, 1e5, 1e8]:
        a = oracle.evaluate_one(o, w, out_R=True, sign=+1)
        b = oracle.evaluate_one(oc, w, out_R=True, sign=-1)
        assert np.max(np.abs(a["P"].conj() - b["P"])) <= 1e-13 * np.max(np.abs(a["P"]))
        for key in ("R", "I", "Delta"):
            assert np.allclose(a[key], b[key], rtol=1e-12, atol=0), key


# ---------------------------------------------------------------- C10: Gram vs explicit residual (a5)
@pytest.mark.parametrize("omega", [10.0, 3e3, 1e6, 1e8])
def test_C10_gram_equals_explicit_residual(c0, omega):
    ops, ex = c0
    out = oracle.evaluate_one(ops, omega)
    res = fullorder.full_residual(ex.K_full, ex.M_full, ex.B0f, ex.B1f, ex.U, out["P"], ops.nu, omega)
    nrm2 = np.array([np.vdot(res[:, i], res[:, i]).real for i in range(3)])
    D = np.zeros((3, 3))
    for i in range(3):
        for j in range(3):
            dij = np.vdot(res[:, i] - res[:, j], res[:, i] - res[:, j]).real
            D[i, j] = ops.alpha ** 3 / (8 * ops.alpha_lb) * (nrm2[i] + nrm2[j] + dij)
    assert np.max(np.abs(out["Delta"] - D) / D) <= 1e-12


# ---------------------------------------------------------------- C11: certificate degeneracies (a5)
def test_C11_certificate_degeneracies(c1ops):
    o = c1ops
    for w in [10.0, 1e4, 1e8]:
        P = solve_reduced(o.K, o.M, o.b0, o.b1, o.nu, w)
        D, n, _ = certificate(P, o.G, o.nu, w, o.alpha, o.alpha_lb)
        assert np.all(D >= 0) and np.array_equal(D, D.T)
        assert np.allclose(np.diag(D), o.alpha ** 3 / (4 * o.alpha_lb) * n, rtol=4 * U, atol=0)
        # homogeneity: doubling the residual (G -> 4G) quadruples Delta
        D4, _, _ = certificate(P, 4 * o.G, o.nu, w, o.alpha, o.alpha_lb)
        assert np.array_equal(D4, 4 * D)
    Dz, nz, _ = certificate(np.zeros((o.r, 3), complex), np.zeros_like(o.G), o.nu, 1e3, o.alpha, o.alpha_lb)
    assert np.array_equal(Dz, np.zeros((3, 3)))          # w = 0 -> 0


def test_certificate_Q_reassociation_matches_explicit(c1ops):
    """Appendix A.2 re-association (what the GPU evaluates) equals the explicit w^H G w form."""
    o = c1ops
    r = o.r
    G = o.G
    Gkk, Gmm = G[6:6 + r, 6:6 + r], G[6 + r:, 6 + r:]
    J = 1j * (G[6:6 + r, 6 + r:] - G[6 + r:, 6:6 + r])
    for w in [10.0, 1e5, 1e8]:
        s = w * o.nu
        P = solve_reduced(o.K, o.M, o.b0, o.b1, o.nu, w)
        _, _, X = certificate(P, G, o.nu, w, o.alpha, o.alpha_lb)
        Q = Gkk + s * J + s * s * Gmm
        for i in range(3):
            for j in range(3):
                d_i = np.array([1.0, w])
                d_j = np.array([1.0, w])
                c = d_i @ G[2 * i:2 * i + 2, 2 * j:2 * j + 2] @ d_j
                li = -(d_i @ (G[2 * i:2 * i + 2, 6:6 + r] + 1j * s * G[2 * i:2 * i + 2, 6 + r:]))
                lj = -(d_j @ (G[2 * j:2 * j + 2, 6:6 + r] + 1j * s * G[2 * j:2 * j + 2, 6 + r:]))
                x = c + li @ P[:, j] + np.conj(lj @ P[:, i]) + np.vdot(P[:, i], Q @ P[:, j])
                assert abs(x - X[i, j]) <= 1e-13 * (abs(X[i, j]) + abs(c) + np.abs(P).max() ** 2 * np.abs(Q).max())


# ---------------------------------------------------------------- C12: selection (a7)
def _grid_with_interval_maxima(lams, per=5, seed=0):
    """Snapshots 1..n+1; 'per' grid points strictly inside each interval with the given maxima."""
    rng = np.random.default_rng(seed)
    snap = np.arange(1, len(lams) + 2, dtype=float)
    om, D, argf = [], [], []
    for n, lam in enumerate(lams):
        pts = snap[n] + (np.arange(per) + 0.5) / per
        vals = rng.random((per, 6)) * lam * 0.9
        k = rng.integers(per)
        vals[k, rng.integers(6)] = lam
        argf.append(len(om) + k)
        om.extend(pts)
        D.extend(vals)
    return np.array(om), np.array(D), snap, argf


def test_C12_spec_golden_examples():
    gd = json.load(open(os.path.join(GOLDEN, "select_spec_examples.json")))
    for case in gd["cases"]:
        om, D, snap, argf = _grid_with_interval_maxima(case["lambda"])
        if case["theta"] is None:
            wnew, idx, Lam, lam = oracle.select(om, D, snap, case["n_star"])
        else:
            wnew, idx, Lam, lam = oracle.select(om, D, snap, 3, theta=case["theta"])
        assert idx == sorted(argf[t] for t in case["chosen_intervals"]), case["cite"]
        assert Lam == max(case["lambda"])


def test_C12_bruteforce_and_conventions():
    rng = np.random.default_rng(3)
    om = np.linspace(1.0, 13.0, 601)
    snap = np.array([1.0, 2.5, 4.0, 7.0, 13.0])
    D = rng.random((len(om), 6))
    wnew, idx, Lam, lam = oracle.select(om, D, snap, 2)
    # Lambda is exactly the maximum of emitted Delta over non-snapshot points
    mask = ~np.isin(om, snap)
    assert Lam == D[mask].max()
    # independent vectorised recomputation of the interval maxima
    n = np.clip(np.searchsorted(snap, om, side="right") - 1, 0, len(snap) - 2)
    for t in range(len(snap) - 1):
        sel = mask & (n == t)
        assert lam[t] == D[sel].max()
    best = sorted(range(4), key=lambda t: (-lam[t], t))[:2]
    exp_idx = []
    for t in best:
        cand = np.where(mask & (n == t))[0]
        exp_idx.append(int(cand[np.argmax(D[cand].max(axis=1))]))
    assert idx == sorted(exp_idx)
    # last interval is closed; points outside [snap0, snapN] are ignored
    om2 = np.array([0.5, 13.5, 12.0, 14.0, 13.0, 11.0])
    D2 = np.array([[9.0] * 6, [8.0] * 6, [7.0] * 6, [9.0] * 6, [1.0] * 6, [2.0] * 6])
    snap2 = np.array([1.0, 12.0, 13.5])
    w2, i2, L2, lam2 = oracle.select(om2, D2, snap2, 1)
    # 0.5, 14 outside; 12.0 and 13.5 equal snapshots -> not candidates
    assert lam2 == [2.0, 1.0] and i2 == [5] and L2 == 2.0 and w2 == [11.0]
    w3, i3, _, _ = oracle.select(om2, D2, snap2, 2)
    assert i3 == [4, 5]
    with pytest.raises(ValueError):
        oracle.select(om2, D2, snap2, 3)


# ---------------------------------------------------------------- N4 epilogues (invariants, coil voltage)
def test_N4_invariants_pins():
    rng = np.random.default_rng(4)
    # isotropic m I -> (m, m, m)
    R6 = np.array([[2.0, 2.0, 2.0, 0, 0, 0]])
    eR, eI = oracle.invariants((R6, R6))
    assert np.array_equal(eR, [[2.0, 2.0, 2.0]])
    # trace and determinant identities, rotation invariance
    for _ in range(5):
        X = rng.standard_normal((3, 3)); T = X + X.T
        Q, _r = np.linalg.qr(rng.standard_normal((3, 3)))
        e1, _ = oracle.invariants((np.array([oracle.to6(T)]), np.array([oracle.to6(T)])))
        e2, _ = oracle.invariants((np.array([oracle.to6(Q @ T @ Q.T)]),) * 2)
        assert abs(e1.sum() - np.trace(T)) < 1e-12 and abs(np.prod(e1) - np.linalg.det(T)) < 1e-11
        assert np.allclose(e1, e2, atol=1e-12)
    # block structure: (1,2)-coupled block + isolated (3,3) entry -> that entry is an eigenvalue
    T = np.array([[1.0, 0.5, 0], [0.5, 2.0, 0], [0, 0, 7.0]])
    e, _ = oracle.invariants((np.array([oracle.to6(T)]),) * 2)
    assert np.isclose(e[0], 7.0).any()


def test_N4_voltage_pins():
    rng = np.random.default_rng(5)
    R6 = rng.standard_normal((4, 6)); I6 = rng.standard_normal((4, 6))
    hx = rng.standard_normal((3, 3)); hm = rng.standard_normal((3, 3))
    V = oracle.coil_voltage(R6, I6, hx, hm)
    assert np.allclose(V, oracle.coil_voltage(R6, I6, hm, hx))           # reciprocity (M symmetric)
    assert np.array_equal(oracle.coil_voltage(0 * R6, 0 * I6, hx, hm), np.zeros((4, 3)))  # M = 0 -> V = 0
    # diagonal M, axis-aligned fields: V = M_kk (h_ms)_k (h_ex)_k
    Rd = np.array([[1.0, 2.0, 3.0, 0, 0, 0]]); Id = np.array([[0.5, 0.0, -1.0, 0, 0, 0]])
    v = oracle.coil_voltage(Rd, Id, [[0, 0, 2.0]], [[0, 0, 3.0]])
    assert v[0, 0] == (3.0 - 1.0j) * 6.0


# ---------------------------------------------------------------- parity metric pins
# The gate's denominators (oracle/parity.py magnitudes(), SURVEY 8(c) "Parity metric") must bound the values they
# normalise (Cauchy-Schwarz in the K_R / M inner products, triangle inequality), and reduce to the value itself in
# the cases where no cancellation is possible -- so a slip that inflates them (a lost sqrt, a dropped factor)
# fails here instead of silently loosening the 1e-10 gate.
def _sweep_cases():
    cases = [("c0", g.make_config0()[0], g.omega_grid(9))]
    for r in (24, 48, 32, 96):
        cases.append((f"r{r}", g.make_operators(r), g.omega_grid(7)))
    cases.append(("pivot-forcing", g.make_pivot_forcing(16, seed=3), g.omega_grid(7)))
    cases.append(("kappa1e8", g.make_illconditioned(8, 1e8, seed=8), g.omega_grid(7)))
    return cases


@pytest.mark.parametrize("name,ops,omegas", _sweep_cases(), ids=lambda x: x if isinstance(x, str) else "")
def test_parity_magnitudes_bound_values(name, ops, omegas):
    from oracle.parity import magnitudes
    for w in omegas:
        o = oracle.evaluate_one(ops, float(w), out_R=True)
        magR, magI, magD = magnitudes(ops, float(w), o["P"])
        R6, I6, D6 = oracle.to6(o["R"]), oracle.to6(o["I"]), oracle.to6(o["Delta"])
        tol = 1e-12
        assert np.all(np.abs(R6) <= magR * (1 + tol)), name
        assert np.all(np.abs(I6) <= magI * (1 + tol)), name
        assert np.all(D6 <= magD * (1 + tol)), name
        K_R = ops.K if ops.K_R is None else ops.K_R
        if np.linalg.eigvalsh(K_R)[0] > 0:
            # diagonal R entries: no cancellation, |R_ii| = (alpha^3/4) p_i^H K_R p_i = mag^R_ii exactly
            assert np.allclose(np.abs(R6[:3]), magR[:3], rtol=1e-13, atol=0), name


def test_parity_magnitudes_equality_cases(c0, c1ops):
    """mag^I_ii = |I_ii| when S = 0 and H = 0 (only the nu p^H M p term; config 0's M is full rank, so p^H M p has
    no cancellation); mag^Delta_ii = 3 Delta_ii when P = 0 and G has non-negative real entries
    (w_i = e_2i + omega e_2i+1 >= 0, so |w|^T |G| |w| = w^T G w = n_i)."""
    from oracle.parity import magnitudes
    o = c0[0]
    ops = g.Operators(**{**o.__dict__, "S": np.zeros((3, 3)), "H": np.zeros_like(o.H)})
    for w in (10.0, 1e4, 1e8):
        ev = oracle.evaluate_one(ops, w, out_R=True)
        _, magI, _ = magnitudes(ops, w, ev["P"])
        assert np.allclose(np.abs(oracle.to6(ev["I"])[:3]), magI[:3], rtol=1e-13, atol=0)
    o = c1ops
    rng = np.random.default_rng(5)
    Wr = rng.uniform(0.0, 1.0, (o.G.shape[0], o.G.shape[0]))
    ops0 = g.Operators(**{**o.__dict__, "b0": np.zeros_like(o.b0), "b1": np.zeros_like(o.b1),
                          "G": (Wr.T @ Wr).astype(np.complex128)})
    for w in (10.0, 1e4, 1e8):
        ev = oracle.evaluate_one(ops0, w, out_R=True)
        _, _, magD = magnitudes(ops0, w, ev["P"])
        D6 = oracle.to6(ev["Delta"])
        assert np.allclose(magD[:3], 3.0 * D6[:3], rtol=1e-13, atol=0)


# ---------------------------------------------------------------- 80-bit adjudication oracle (oracle/extended.py)
def test_extended_oracle_matches_fp64_when_well_conditioned(c1ops):
    from oracle.extended import evaluate_one_ld
    from oracle.parity import errors
    for w in (10.0, 3.7e3, 2.2e6, 1e8):
        e = evaluate_one_ld(c1ops, w)
        o = oracle.evaluate_one(c1ops, w, out_R=True)
        eR, eI, eD = errors(c1ops, w, e["R6"], e["I6"], e["D6"], oracle.to6(o["R"]), oracle.to6(o["I"]),
                            oracle.to6(o["Delta"]))
        assert eR.max() <= 1e-11 and eI.max() <= 1e-11 and eD.max() <= 1e-9


def test_extended_oracle_solve_residual_and_scalar_closed_form():
    from oracle.extended import CLD, evaluate_one_ld, solve_ld
    ops = g.make_illconditioned(8, 1e8, seed=8)
    s = 1e7 * ops.nu
    A = ops.K.astype(CLD) + CLD(1j) * CLD(s) * ops.M.astype(CLD)
    B = ops.b0.astype(CLD) + CLD(1e7) * ops.b1.astype(CLD)
    X = solve_ld(A, B)
    res = np.abs(A @ X - B).max() / (np.abs(A).max() * np.abs(X).max())
    assert res < 1e-17  # long double unit roundoff 5.4e-20, r = 8
    # r = 1 closed form (pin C2 in long double): p = (b0 + w b1)/(k + i w nu m)
    k, m, b0, b1, w = 3.0, 0.5, 1 + 2j, -0.25 + 1j, 1e3
    one = g.Operators(K=np.array([[k + 0j]]), M=np.array([[m + 0j]]), b0=np.full((1, 3), b0),
                      b1=np.full((1, 3), b1), N0=np.eye(3), S=np.zeros((3, 3)), H=np.zeros((3, 1), complex),
                      G=np.eye(8, dtype=complex), nu=0.1, alpha=1.0, alpha_lb=1.0)
    e = evaluate_one_ld(one, w)
    p = (b0 + w * b1) / (k + 1j * w * 0.1 * m)
    assert abs(e["P"][0, 0] - p) <= 1e-15 * abs(p)
    assert abs(e["R6"][0] - (-0.25 * k * abs(p) ** 2)) <= 1e-15 * 0.25 * k * abs(p) ** 2
