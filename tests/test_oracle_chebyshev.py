"""Pins for oracle/chebyshev.py (CPU only).

Pinned against: the Chebyshev polynomial contract e_p = T_p((theta-B)/delta)/T_p(theta/delta) e_0
(numpy.polynomial.chebyshev on the eigen-decomposition);
Prop. prop:errorbound; Thm thm:convergence asymptotics
(PAPER.md:465-510); Algorithm 1 vs all 83 NC2 cells of Tables 3, 4 and 8
(PAPER.md:788-803, 832-847, 962-966); the printed Table 2 real columns (soft);
P_NC -> exact P_alpha^{-1} as the budget grows; c = 0 exactness.
"""
import json
import math
import os

import numpy as np
import numpy.polynomial.chebyshev as npch
import pytest

import synth
from oracle import chebyshev as ch
from oracle import circulant as circ
from oracle import operator as op
from oracle import paper

HERE = os.path.dirname(__file__)
TABLES = json.load(open(os.path.join(HERE, "golden", "paper_nc2_tables.json")))
SCAL = json.load(open(os.path.join(HERE, "golden", "paper_scalars.json")))


def _w(shape=(1, 5, 6), seed=0, c=None):
    rng = np.random.default_rng(seed)
    nz, ny, nx = shape
    return op.Weights(shape, 0.6 / nx ** 2 if c is None else c,
                      np.exp(0.3 * rng.standard_normal((nz, ny, nx - 1))),
                      np.exp(0.3 * rng.standard_normal((nz, ny - 1, nx))),
                      np.exp(0.3 * rng.standard_normal((nz - 1, ny, nx))))


def _Tp(p, z):
    return npch.chebval(z, [0] * p + [1])


@pytest.mark.parametrize("lam", [0.63, -0.4, 0.3 - 0.5j, -0.2 + 0.33j])
@pytest.mark.parametrize("p", [1, 2, 5, 9])
def test_polynomial_contract(lam, p):
    w = _w()
    A = op.dense_A(w)
    mu, X = np.linalg.eigh(A)
    mu_min, mu_max = 1.0, op.gershgorin_max(w)
    theta = 0.5 * (mu_max + mu_min) - lam
    delta = 0.5 * (mu_max - mu_min)
    b = np.random.default_rng(1).standard_normal(w.N) + 0.5j * np.random.default_rng(2).standard_normal(w.N)
    B = A - lam * np.eye(w.N)
    xstar = np.linalg.solve(B, b)
    xp = ch.ci_solve(lambda v: (B @ v.ravel()).reshape(v.shape), b, theta, delta, p)
    xi = mu - lam                                            # eigenvalues of B
    omega = _Tp(p, (theta - xi) / delta) / _Tp(p, theta / delta)
    ep = X @ (omega * (X.T @ xstar))                         # e_p = Omega_p(B) e_0, e_0 = x*
    assert np.linalg.norm((xstar - xp) - ep) <= 1e-12 * np.linalg.norm(xstar)


@pytest.mark.parametrize("lam", [0.5, -0.5, 0.4 + 0.3j])
def test_prop_errorbound_every_p(lam):
    w = _w((1, 6, 5), seed=3)
    A = op.dense_A(w)
    mu = np.linalg.eigvalsh(A)
    theta = 0.5 * (mu.max() + mu.min()) - lam
    delta = 0.5 * (mu.max() - mu.min())
    B = A - lam * np.eye(w.N)
    b = np.random.default_rng(4).standard_normal(w.N).astype(complex)
    xstar = np.linalg.solve(B, b)
    for p in range(1, 25):
        xp = ch.ci_solve(lambda v: B @ v, b, theta, delta, p)
        bound = 1.0 / abs(_Tp(p, theta / delta))           # |T_p((xi1+xiN)/(xi1-xiN))|^{-1}
        assert np.linalg.norm(xstar - xp) / np.linalg.norm(xstar) <= bound * (1 + 1e-9)


@pytest.mark.parametrize("k", [0, 1, 2, 3])
def test_thm_convergence_asymptotic_factor(k):
    """Late geometric-mean error reduction <= sigma(Re Lambda_k) + 0.01 (Thm 3.6) with
    exact extreme eigenvalues (north_star oracle item 5)."""
    w = _w((1, 10, 10), seed=5, c=3.0 / 100)
    A = op.dense_A(w)
    mu = np.linalg.eigvalsh(A)
    ell, alpha = 8, 0.5
    lam = circ.shifts(ell, alpha)[k]
    theta = 0.5 * (mu.max() + mu.min()) - lam
    delta = 0.5 * (mu.max() - mu.min())
    B = A - lam * np.eye(w.N)
    b = np.random.default_rng(6).standard_normal(w.N).astype(complex)
    xstar = np.linalg.solve(B, b)
    e = [np.linalg.norm(xstar - ch.ci_solve(lambda v: B @ v, b, theta, delta, p)) for p in (20, 40)]
    rate = (e[1] / e[0]) ** (1.0 / 20)
    sigma = ch.sigma_bound(mu.min(), mu.max(), lam.real)
    assert rate <= sigma + 0.01
    assert sigma < 1.0


def test_sigma_examples_and_pstar_vs_table2():
    lo, hi = paper.bounds(100, 10)
    assert lo == pytest.approx(1.04934, abs=5e-6) and hi == pytest.approx(204.97, abs=5e-3)
    kap = (hi - 1.0) / (lo - 1.0)
    assert kap == pytest.approx(4133.6, abs=0.1)
    assert ch.sigma_bound(lo, hi, 1.0) == pytest.approx(0.9694, abs=1e-4)
    assert ch.sigma_bound(lo, hi, -1.0) == pytest.approx(0.8186, abs=1e-4)
    # Thm 3.1 a-priori count vs the measured 463 of Table 2: within 1%
    ps = math.ceil(ch.p_star(lo - 1.0, hi - 1.0, 1e-6))
    assert ps == 467 and abs(ps - SCAL["table2_1e-6"]["lambda1"]) / 463 < 0.01
    # monotone: sigma increases with Re lambda (bullet after Thm 3.6)
    s = [ch.sigma_bound(lo, hi, r) for r in (-1, -0.5, 0, 0.5, 1)]
    assert all(a < b for a, b in zip(s, s[1:]))


def test_table2_real_columns_soft():
    """CI iterations to 1e-6 on the paper operator (n_x=100, ell=10, alpha=1): lambda=1 -> 463,
    lambda=-1 -> 72. Soft pin +-2% (reading R13: the complex columns do not
    reproduce with textbook CI; the real ones do)."""
    A = paper.sparse_A(100, 10)
    lo, hi = paper.bounds(100, 10)
    b = np.random.default_rng(0).standard_normal(A.shape[0])
    out = {}
    for lam in (1.0, -1.0):
        theta = 0.5 * (hi + lo) - lam
        delta = 0.5 * (hi - lo)
        out[lam] = ch.ci_iterations_to_tol(lambda v, lam=lam: A @ v - lam * v, b, theta, delta,
                                           1e-6, 2000)
    assert abs(out[1.0] - 463) <= 0.02 * 463
    assert abs(out[-1.0] - 72) <= 0.02 * 72 + 1


def _cells():
    t3, t4, t8 = TABLES["table3"], TABLES["table4"], TABLES["table8"]
    for akey, alpha in (("alpha_1", 1.0), ("alpha_0.01", 0.01)):
        for nx, row in t3[akey].items():
            for eta, (outer, tot) in zip(t3["eta"], row):
                yield ("T3", int(nx), t3["ell"], alpha, eta, outer, tot)
        for ell, row in t4[akey].items():
            for eta, (outer, tot) in zip(t4["eta"], row):
                yield ("T4", t4["nx"], int(ell), alpha, eta, outer, tot)
    for nx, (outer, tot) in t8["cells"].items():
        yield ("T8", int(nx), t8["ell"], t8["alpha"], t8["eta"], outer, tot)


def test_algorithm1_reproduces_all_nc2_cells():
    cells = list(_cells())
    assert len(cells) == 83
    bad = []
    for tab, nx, ell, alpha, eta, outer, tot in cells:
        assert tot % outer == 0
        lo, hi = paper.bounds(nx, ell)
        alloc = ch.allocate(ell, lo, hi, alpha, ell * nx * eta, "nc2")
        if sum(alloc) != tot // outer - ell:
            bad.append((tab, nx, ell, alpha, eta, sum(alloc), tot // outer - ell))
        # conjugate pairs equal; larger Re(lambda) gets >= iterations
        assert all(alloc[k] == alloc[ell - k] for k in range(1, ell))
        assert all(alloc[k] >= alloc[k + 1] for k in range(ell // 2))
    assert not bad, bad


def test_algorithm1_worked_example_and_headline():
    lo, hi = paper.bounds(100, 10)
    assert ch.allocate(10, lo, hi, 1.0, 200, "nc2") == [60, 27, 15, 11, 9, 9, 9, 11, 15, 27]
    assert ch.allocate(10, 1.0, 32.14052450955844, 1e-4, 80, "nc2") == [9, 9, 8, 7, 6, 6, 6, 7, 8, 9]
    assert ch.allocate(10, lo, hi, 1.0, 200, "nc1", 20) == [20] * 10
    # NC1 accounting of Table 3: 9840/164 = ell + ell*floor(n_x eta)
    g = SCAL["nc1_budget"]
    assert g["total"] // g["outer"] == g["ell"] * (1 + g["per_block"])


@pytest.mark.parametrize("ell,alpha", [(4, 0.3), (6, 1e-2)])
def test_nc_converges_to_exact(ell, alpha):
    w = _w((1, 4, 5), seed=7)
    mu_max = op.gershgorin_max(w)
    r = np.random.default_rng(8).standard_normal((ell,) + w.shape)
    z = circ.exact_apply(w, r, ell, alpha)
    errs = []
    for k in (5, 10, 20, 40, 80):
        zn = ch.nc_apply(w, r, ell, alpha, 1.0, mu_max, [k] * ell)
        errs.append(np.linalg.norm(zn - z) / np.linalg.norm(z))
    assert all(b < a for a, b in zip(errs, errs[1:]))
    assert errs[-1] < 1e-9


def test_c_zero_nc_is_exact():
    w = _w((1, 4, 4), c=0.0)
    ell, alpha = 10, 1e-4
    r = np.random.default_rng(9).standard_normal((ell,) + w.shape)
    z = ch.nc_apply(w, r, ell, alpha, 1.0, op.gershgorin_max(w), [1] * ell)
    zd = np.linalg.solve(circ.dense_P_alpha(op.dense_A(w), ell, alpha), r.ravel())
    assert np.linalg.norm(z.ravel() - zd) <= 1e-12 * np.linalg.norm(zd) * circ.gamma_condition(ell, alpha)


def test_paper_nc1_golden_is_self_consistent():
    """The typed NC1 cells of Tables 3/4 (tests/golden/paper_nc1_tables.json): P_NC1 spends
    ell (calA) + ell * n_x * eta (inner) matvecs per outer iteration (Table 1),
    so every printed total equals its iteration count times that -- a check on every cell."""
    d = json.load(open(os.path.join(HERE, "golden", "paper_nc1_tables.json")))
    for tab in ("table3", "table4"):
        T = d[tab]
        for a in ("alpha_1", "alpha_0.01"):
            for key, cells in T[a].items():
                ell = T["ell"] if tab == "table3" else int(key)
                nx = int(key) if tab == "table3" else T["nx"]
                for eta, (its, mv) in zip(T["eta"], cells):
                    assert its * (ell + ell * round(nx * eta)) == mv, (tab, a, key, eta)


@pytest.mark.parametrize("method,k", [("nc1", 6), ("nc2", 8)])
def test_nc_apply_f32_is_nc_apply_to_single_precision(method, k):
    """The mixed-precision variant (fp32 recurrence) agrees with the fp64 nc_apply to fp32
    rounding (unit 6e-8) amplified by at most kappa(Gamma_alpha) through the inverse transform
    (reading R18), and is NOT bit-identical (it is fp32)."""
    p = synth.make_problem("headline", shape=(1, 20, 17))
    w = op.weights(p)
    mu = op.gershgorin_max(w)
    al = ch.allocate(p.ell, 1.0, mu, p.alpha, p.ell * k, method, k)
    r = np.random.default_rng(8).standard_normal((p.ell,) + p.shape)
    z64 = ch.nc_apply(w, r, p.ell, p.alpha, 1.0, mu, al)
    z32 = ch.nc_apply_f32(w, r, p.ell, p.alpha, 1.0, mu, al)
    e = np.linalg.norm(z32 - z64) / np.linalg.norm(z64)
    assert 1e-9 < e < 6e-8 * circ.gamma_condition(p.ell, p.alpha)
