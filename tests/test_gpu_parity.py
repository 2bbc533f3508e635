"""GPU parity: the CUDA path (through the C ABI) vs the oracle on identical seeded inputs.

Bars (BASELINE.json north_star): relative 2-norm <= 1e-12 per calA or preconditioner apply,
<= 1e-9 on the GMRES solution, iteration counts equal within +-1. Integer outputs (the
NC2 allocation) are compared bit-exactly. Sizes span several CTA tiles with ragged tails;
the full-size headline is checked against oracle values stored by
scripts/make_oracle_golden.py (oracle-only) and by properties that hold at any size.
"""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import synth  # noqa: E402
from oracle import chebyshev as ch  # noqa: E402
from oracle import circulant as circ  # noqa: E402
from oracle import gmres as og  # noqa: E402
from oracle import operator as op  # noqa: E402

HERE = os.path.dirname(__file__)


def _solver(p, max_krylov=64):
    from paper_2506_03947_b200 import from_problem
    return from_problem(p, max_krylov=max_krylov)


def _dev(a, ell):
    return torch.from_numpy(np.ascontiguousarray(a).reshape(ell, -1)).cuda()


def _rel(a, b):
    a = np.asarray(a).ravel()
    b = np.asarray(b).ravel()
    return np.linalg.norm(a - b) / np.linalg.norm(b)


CASES = [
    ("1d", {}),
    ("2d256", dict(shape=(1, 53, 37))),
    ("2d256", dict(shape=(1, 2, 2), ell=2)),
    ("headline", dict(shape=(1, 130, 67))),
    ("2d256", dict(n=256, alpha=1e-4)),
    ("3d", dict(shape=(9, 13, 11))),
    ("3d", dict(shape=(17, 17, 17), ell=4)),
    # even nx, ragged 256-column / 8-row tiles of k_matvec_tile (516 = 2 x 256 + 4)
    ("headline", dict(shape=(1, 131, 516))),
    ("2d256", dict(shape=(1, 9, 600), ell=4)),
]


_MATVEC_BITS = """
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import synth
from paper_2506_03947_b200 import from_problem
p = synth.make_problem("headline", shape=(1, 131, 516))
s = from_problem(p, max_krylov=8)
x = np.random.default_rng(7).standard_normal((p.ell,) + p.shape)
y = s.matvec(torch.from_numpy(x.reshape(p.ell, -1)).cuda()).cpu().numpy()
np.save({out!r}, y)
"""


def test_matvec_tile_bit_identical_to_register_kernel(tmp_path):
    """k_matvec_tile (TMA-staged tiles, AAC_MATVEC_TILE=1) performs stencil_sv's operations in the
    same order: its result equals k_matvec's (the default, a fresh process each) bit for bit."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for flag in ("1", "0"):
        out = str(tmp_path / f"y{flag}.npy")
        r = subprocess.run([sys.executable, "-c", _MATVEC_BITS.format(root=root, out=out)], capture_output=True,
                           text=True, timeout=300, env={**os.environ, "AAC_MATVEC_TILE": flag})
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(out))
    assert np.array_equal(outs[0], outs[1])


_MATVEC_BITS_KW = """
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import synth
from paper_2506_03947_b200 import from_problem
p = synth.make_problem({name!r}, **{kw!r})
s = from_problem(p, max_krylov=8)
x = np.random.default_rng(7).standard_normal((p.ell,) + p.shape)
y = s.matvec(torch.from_numpy(x.reshape(p.ell, -1)).cuda()).cpu().numpy()
np.save({out!r}, y)
"""


@pytest.mark.parametrize("name,kw,ry", [
    ("headline", dict(shape=(1, 131, 516)), ""), ("headline", dict(shape=(1, 131, 516)), "3"),
    ("headline", dict(shape=(1, 130, 67 + 1)), "1"), ("2d256", dict(shape=(1, 9, 600), ell=4), "16"),
    ("2d256", dict(shape=(1, 2, 2), ell=2), ""), ("2d256", dict(shape=(1, 41, 40), ell=12, alpha=0.3), "5"),
    ("headline", dict(shape=(1, 64, 64), c=0.0), ""),
])
def test_matvec_rows_bit_identical_to_register_kernel(tmp_path, name, kw, ry):
    """k_matvec_rows (row-marching, 2D with even nx, opt-in AAC_MATVEC_ROWS=1; AAC_MATVEC_RY rows per thread,
    ragged last chunks) performs stencil_sv's operations in the same order: its result equals
    k_matvec's (AAC_MATVEC_ROWS=0) bit for bit, a fresh process each."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for flag in ("1", "0"):
        out = str(tmp_path / f"y{flag}.npy")
        env = {**os.environ, "AAC_MATVEC_ROWS": flag}
        if ry:
            env["AAC_MATVEC_RY"] = ry
        r = subprocess.run([sys.executable, "-c", _MATVEC_BITS_KW.format(root=root, name=name, kw=kw, out=out)],
                           capture_output=True, text=True, timeout=300, env=env)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(out))
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("name,kw", CASES)
def test_matvec_parity(name, kw):
    p = synth.make_problem(name, **kw)
    s = _solver(p)
    w = op.weights(p)
    assert s.mu_max == pytest.approx(op.gershgorin_max(w), rel=1e-14)
    x = np.random.default_rng(7).standard_normal((p.ell,) + p.shape)
    y = s.matvec(_dev(x, p.ell)).cpu().numpy()
    assert _rel(y, op.apply_allatonce(w, x)) <= 1e-12
    s.close()


PRE = [
    ("1d", {}, "nc1", 10), ("1d", {}, "nc2", 10), ("1d", {}, "nc1", 1),
    ("2d256", dict(shape=(1, 53, 37)), "nc1", 5), ("2d256", dict(shape=(1, 53, 37)), "nc2", 5),
    ("2d256", dict(shape=(1, 53, 37), alpha=1e-4), "nc1", 2),
    ("2d256", dict(shape=(1, 41, 40), ell=2), "nc1", 4),
    ("2d256", dict(shape=(1, 41, 40), ell=16, alpha=0.3), "nc2", 6),
    ("headline", dict(shape=(1, 130, 67)), "nc2", 8),
    ("headline", dict(shape=(1, 64, 64), c=0.0), "nc2", 8),
    ("3d", dict(shape=(9, 13, 11)), "nc1", 10), ("3d", dict(shape=(9, 13, 11)), "nc2", 3),
]


@pytest.mark.parametrize("name,kw,method,k", PRE)
def test_precond_parity(name, kw, method, k):
    p = synth.make_problem(name, **kw)
    s = _solver(p)
    w = op.weights(p)
    mu = op.gershgorin_max(w)
    al = ch.allocate(p.ell, 1.0, mu, p.alpha, p.ell * k, method, k)
    assert s.allocation(method, k) == al                      # integer decision: bit-exact
    r = np.random.default_rng(3).standard_normal((p.ell,) + p.shape)
    z = s.precond_apply(method, k, _dev(r, p.ell)).cpu().numpy()
    zo = ch.nc_apply(w, r, p.ell, p.alpha, 1.0, mu, al)
    assert _rel(z, zo) <= 1e-12
    s.close()


def test_precond_c_zero_equals_exact_P_alpha():
    """c = 0: every block is solved exactly at p = 1, so P_NC^{-1} = P_alpha^{-1}."""
    p = synth.make_problem("headline", shape=(1, 12, 9), c=0.0)
    s = _solver(p)
    w = op.weights(p)
    r = np.random.default_rng(4).standard_normal((p.ell,) + p.shape)
    z = s.precond_apply("nc2", 8, _dev(r, p.ell)).cpu().numpy()
    zd = np.linalg.solve(circ.dense_P_alpha(op.dense_A(w), p.ell, p.alpha), r.ravel())
    assert _rel(z, zd) <= 1e-12 * circ.gamma_condition(p.ell, p.alpha)
    s.close()


GM = [
    ("1d", {}, None, None),
    # BASELINE.json configs[1]: 256^2, alpha in {1e-2, 1e-4} x k in {5, 20} -- all four pairs
    ("2d256", dict(n=256), "nc1", 5),
    ("2d256", dict(n=256), "nc1", 20),
    ("2d256", dict(n=256, alpha=1e-4), "nc1", 5),
    ("2d256", dict(n=256, alpha=1e-4), "nc1", 20),
    ("headline", dict(n=256), "nc2", 8),
    ("headline", dict(shape=(1, 100, 73)), "nc1", 8),
    ("3d", dict(shape=(16, 16, 16)), "nc1", 10),
    # 64^3, ell = 12: large enough that k_arnoldi streams every basis vector of a tile in one
    # CTA (ng = 1), as at the full 256^3 size of configs[4] (~25 s of oracle)
    ("3d", dict(n=64), "nc1", 10),
]


def _oracle_gmres(p, method, k, maxit=200):
    w = op.weights(p)
    mu = op.gershgorin_max(w)
    al = ch.allocate(p.ell, 1.0, mu, p.alpha, p.ell * k, method, k)
    return og.fgmres(lambda x: op.apply_allatonce(w, x),
                     lambda r: ch.nc_apply(w, r, p.ell, p.alpha, 1.0, mu, al), p.b, p.rtol, maxit)


@pytest.mark.parametrize("name,kw,method,k", GM)
def test_gmres_parity(name, kw, method, k):
    p = synth.make_problem(name, **kw)
    method = method or p.method
    k = k or p.k
    s = _solver(p, max_krylov=80)
    x, info = s.gmres(method, k, _dev(p.b, p.ell), rtol=p.rtol, maxit=80)
    ro = _oracle_gmres(p, method, k, 80)
    assert info["converged"] == 1 and ro.converged
    assert abs(info["iters"] - ro.iters) <= 1
    assert _rel(x.cpu().numpy(), ro.x) <= 1e-9
    assert info["relres_true"] <= 1.5 * p.rtol
    # paper-unit accounting (Table 1): ell + sum(alloc) per outer iteration
    al = s.allocation(method, k)
    assert info["matvecs_paper_units"] == info["iters"] * (p.ell + sum(al))
    s.close()


@pytest.mark.parametrize("name,kw,method,k", [("headline", dict(shape=(1, 130, 67)), "nc2", 8),
                                              ("2d256", dict(n=256), "nc1", 5),
                                              ("3d", dict(shape=(16, 16, 16)), "nc1", 10),
                                              ("saddle", dict(shape=(1, 48, 40)), "sp", 8)])
def test_gmres_one_reduce_parity(monkeypatch, name, kw, method, k):
    """One-reduce Arnoldi (AAC_GMRES_1R=1, the default on several ranks): the
    norm of each new basis vector comes from the Gram column of the projection pass, so every
    step does one reduction. Same counts (+-1) and solutions (1e-9) as the oracle's literal CGS2,
    and iterate-for-iterate the same as the two-reduction path at a forced equal m."""
    from oracle import saddle
    monkeypatch.setenv("AAC_GMRES_1R", "1")
    p = synth.make_problem(name, **kw)
    s = _solver(p, max_krylov=60)
    x, info = s.gmres(method, k, _dev(p.b, p.ell), rtol=p.rtol, maxit=60)
    if method == "sp":
        w = op.weights(p)
        lev = saddle.hierarchy(w)
        ro = og.fgmres(lambda v: op.apply_allatonce(w, v),
                       lambda r: saddle.sp_apply(w, r, p.ell, p.alpha, k, lev), p.b, p.rtol, 60)
    else:
        ro = _oracle_gmres(p, method, k, 60)
    assert info["converged"] == 1 and abs(info["iters"] - ro.iters) <= 1
    assert _rel(x.cpu().numpy(), ro.x) <= 1e-9
    assert info["relres_true"] <= 1.5 * p.rtol
    xm, im = s.gmres(method, k, _dev(p.b, p.ell), rtol=0.0, maxit=6)
    s.close()
    monkeypatch.setenv("AAC_GMRES_1R", "0")
    s2 = _solver(p, max_krylov=60)
    x2, i2 = s2.gmres(method, k, _dev(p.b, p.ell), rtol=0.0, maxit=6)
    assert im["iters"] == i2["iters"] == 6
    assert _rel(xm.cpu().numpy(), x2.cpu().numpy()) <= 1e-12
    s2.close()


def test_gmres_equal_iteration_count_agreement():
    """Forced equal m (rtol = 0, maxit = m): GPU and oracle iterates agree far below 1e-9."""
    p = synth.make_problem("2d256", shape=(1, 40, 45))
    s = _solver(p, max_krylov=8)
    x, info = s.gmres("nc1", 5, _dev(p.b, p.ell), rtol=0.0, maxit=6)
    ro = _oracle_gmres(p, "nc1", 5, 6)
    assert info["iters"] == 6 and info["converged"] == 0
    assert _rel(x.cpu().numpy(), ro.x) <= 1e-11
    s.close()


@pytest.mark.parametrize("rhs,expect", [("b1", 1), ("all", 2)])
def test_gmres_c_zero_exact_counts(rhs, expect):
    p = synth.make_problem("headline", n=16, c=0.0, rhs=rhs)
    s = _solver(p, max_krylov=8)
    x, info = s.gmres("nc2", 8, _dev(p.b, p.ell), rtol=1e-10, maxit=8)
    assert info["iters"] == expect and info["converged"] == 1
    s.close()


def test_gmres_host_path_matches_device_path():
    p = synth.make_problem("headline", shape=(1, 48, 40))
    s = _solver(p, max_krylov=40)
    xd, info_d = s.gmres("nc2", 8, _dev(p.b, p.ell), rtol=p.rtol, maxit=40)
    xh, info_h = s.gmres_host("nc2", 8, p.b.reshape(p.ell, -1), rtol=p.rtol, maxit=40)
    assert info_d["iters"] == info_h["iters"]
    assert np.array_equal(xd.cpu().numpy(), xh)                # deterministic reductions
    s.close()


def test_gmres_host_batch_matches_device_path():
    """aac_gmres_host_batch (copies overlapped with the solves, two device slots reused across
    five systems) returns, per system, exactly what aac_gmres returns on the device."""
    p = synth.make_problem("headline", shape=(1, 48, 40))
    s = _solver(p, max_krylov=40)
    rng = np.random.default_rng(7)
    bs = [p.b.reshape(p.ell, -1)] + [rng.standard_normal((p.ell, p.N)) for _ in range(4)]
    xs, infos = s.gmres_host_batch("nc2", 8, bs, rtol=p.rtol, maxit=40)
    assert len(xs) == len(infos) == 5
    for b, x, info in zip(bs, xs, infos):
        xd, info_d = s.gmres("nc2", 8, torch.from_numpy(np.ascontiguousarray(b)).cuda(), rtol=p.rtol, maxit=40)
        assert info["iters"] == info_d["iters"] and info["converged"] == 1
        assert np.array_equal(xd.cpu().numpy(), x)
    # a repeated output buffer: the copies out are ordered, the last system wins
    xo = np.empty((p.ell, p.N))
    xs2, _ = s.gmres_host_batch("nc2", 8, bs[:3], [xo] * 3, rtol=p.rtol, maxit=40)
    assert np.array_equal(xo, xs[2])
    assert s.gmres_host_batch("nc2", 8, [])[0] == []
    # maxit reached on every system: AAC_ENOCONV is a completed call, each x is the last iterate
    xs3, infos3 = s.gmres_host_batch("nc2", 8, bs[:2], rtol=p.rtol, maxit=3)
    for b, x, info in zip(bs[:2], xs3, infos3):
        xd, info_d = s.gmres("nc2", 8, torch.from_numpy(np.ascontiguousarray(b)).cuda(), rtol=p.rtol, maxit=3)
        assert info["iters"] == info_d["iters"] == 3 and info["converged"] == 0
        assert np.array_equal(xd.cpu().numpy(), x)
    s.close()


def test_gmres_zero_rhs_and_enoconv():
    p = synth.make_problem("headline", shape=(1, 20, 20))
    s = _solver(p, max_krylov=4)
    x, info = s.gmres("nc2", 8, torch.zeros(p.ell, p.N, dtype=torch.float64, device="cuda"), maxit=4)
    assert info["iters"] == 0 and info["converged"] == 1 and not x.abs().max().item()
    x, info = s.gmres("nc1", 1, _dev(p.b, p.ell), rtol=1e-14, maxit=3)
    assert info["iters"] == 3 and info["converged"] == 0
    s.close()


def test_alpha_at_or_above_mu_min_pow_ell_is_rejected():
    """Neumann: mu_min = 1 exactly, so alpha >= 1 makes P_alpha singular (Lemma lemma:Zalpha)
    -- setup accepts it (the paper's Dirichlet operator allows alpha = 1), every apply refuses."""
    from paper_2506_03947_b200 import AacError
    p = synth.make_problem("headline", shape=(1, 8, 8), alpha=1.0)
    s = _solver(p, max_krylov=4)
    r = _dev(np.ones((p.ell, p.N)), p.ell)
    for m in ("nc1", "nc2", "sp"):
        with pytest.raises(AacError, match="Lemma"):
            s.precond_apply(m, 2, r)
    with pytest.raises(AacError, match="Lemma"):
        s.gmres("nc2", 2, r, maxit=4)
    s.close()


def test_bad_arguments_raise():
    from paper_2506_03947_b200 import AacError
    p = synth.make_problem("headline", shape=(1, 8, 8))
    s = _solver(p, max_krylov=4)
    r = _dev(np.ones((p.ell, p.N)), p.ell)
    with pytest.raises(AacError):
        s.precond_apply("nc1", 0, r)
    with pytest.raises(AacError):
        s.gmres("nc1", 2, r, maxit=5)                           # maxit > max_krylov
    s.close()


# ---------------------------------------------------------------- full-size headline
def test_headline_full_size_apply_parity():
    """calA and P_NC2 applies at N = 1024^2, ell = 10 (the bench launch configuration)."""
    p = synth.make_problem("headline")
    s = _solver(p, max_krylov=4)
    w = op.weights(p)
    mu = op.gershgorin_max(w)
    al = ch.allocate(p.ell, 1.0, mu, p.alpha, p.ell * p.k, "nc2")
    assert al == [9, 9, 8, 7, 6, 6, 6, 7, 8, 9] and s.allocation("nc2", p.k) == al
    r = np.random.default_rng(11).standard_normal((p.ell,) + p.shape)
    assert _rel(s.matvec(_dev(r, p.ell)).cpu().numpy(), op.apply_allatonce(w, r)) <= 1e-12
    z = s.precond_apply("nc2", p.k, _dev(r, p.ell)).cpu().numpy()
    assert _rel(z, ch.nc_apply(w, r, p.ell, p.alpha, 1.0, mu, al)) <= 1e-12
    s.close()


def test_headline_full_size_gmres_vs_stored_oracle():
    g = json.load(open(os.path.join(HERE, "golden", "oracle_headline.json")))
    p = synth.make_problem("headline")
    s = _solver(p, max_krylov=40)
    x, info = s.gmres("nc2", p.k, _dev(p.b, p.ell), rtol=p.rtol, maxit=40)
    assert abs(info["iters"] - g["iters"]) <= 1 and info["converged"] == 1
    assert info["relres_true"] <= 1.5 * p.rtol
    xs = x.cpu().numpy().ravel()
    idx = np.array(g["sample_idx"])
    ref = np.array(g["sample_x"])
    assert np.linalg.norm(xs[idx] - ref) <= 1e-9 * np.linalg.norm(ref)
    assert np.linalg.norm(xs) == pytest.approx(g["x_norm"], rel=1e-9)
    s.close()


def test_headline_full_size_gmres_full_vector_vs_oracle():
    """The full headline solve (N = 1024^2, ell = 10, NC2 k = 8) element by element against an
    oracle FGMRES run in this test (~95 s of CPU): counts +-1, the whole x to 1e-9, and the
    forced-equal-m iterate (rtol = 0, maxit = the oracle's count) far below that."""
    p = synth.make_problem("headline")
    ro = _oracle_gmres(p, "nc2", p.k, 40)
    s = _solver(p, max_krylov=40)
    x, info = s.gmres("nc2", p.k, _dev(p.b, p.ell), rtol=p.rtol, maxit=40)
    assert ro.converged and info["converged"] == 1
    assert abs(info["iters"] - ro.iters) <= 1
    assert _rel(x.cpu().numpy(), ro.x) <= 1e-9
    xm, im = s.gmres("nc2", p.k, _dev(p.b, p.ell), rtol=0.0, maxit=ro.iters)
    assert im["iters"] == ro.iters
    assert _rel(xm.cpu().numpy(), ro.x) <= 1e-11
    s.close()


# ---------------------------------------------------------------- saddle-point inner solver (SP)
SP_CASES = [
    ("saddle", dict(shape=(1, 40, 36)), 8),
    ("saddle", dict(shape=(1, 37, 53), ell=4, alpha=1e-2), 3),
    ("2d256", dict(shape=(1, 24, 20), ell=12, alpha=0.3), 5),
    ("1d", {}, 4),
    ("3d", dict(shape=(12, 10, 9), ell=6), 3),
    # several strips / row chunks of the fused 2D level kernels (sp_fused.cuh), odd and even nx
    ("saddle", dict(shape=(1, 261, 517), ell=4, alpha=1e-2), 3),
    ("saddle", dict(shape=(1, 200, 600), ell=6), 2),
]


@pytest.mark.parametrize("name,kw,k", SP_CASES)
def test_sp_precond_parity(name, kw, k):
    from oracle import saddle
    p = synth.make_problem(name, **kw)
    s = _solver(p)
    w = op.weights(p)
    r = np.random.default_rng(5).standard_normal((p.ell,) + p.shape)
    z = s.precond_apply("sp", k, _dev(r, p.ell)).cpu().numpy()
    zo = saddle.sp_apply(w, r, p.ell, p.alpha, k)
    assert _rel(z, zo) <= 1e-12
    s.close()


_SP_VARIANT = """
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import synth
from oracle import operator as op, saddle
from paper_2506_03947_b200 import from_problem
p = synth.make_problem("saddle", shape=(1, 37, 53), ell=4, alpha=1e-2)
s = from_problem(p, max_krylov=8)
w = op.weights(p)
r = np.random.default_rng(6).standard_normal((p.ell,) + p.shape)
z = s.precond_apply("sp", 3, torch.from_numpy(r.reshape(p.ell, -1)).cuda()).cpu().numpy()
zo = saddle.sp_apply(w, r, p.ell, p.alpha, 3).reshape(p.ell, -1)
e = np.linalg.norm(z - zo) / np.linalg.norm(zo)
assert e <= 1e-12, e
print("ok", e)
"""


@pytest.mark.parametrize("env", [dict(AAC_SP_ROW2D="0", AAC_SP_FUSED="0"), dict(AAC_SP_PAIR="0", AAC_SP_FUSED="0"),
                                 dict(AAC_SP_TAIL="0"), dict(AAC_SP_FUSED="0")])
def test_sp_kernel_variants_parity(env):
    """The non-default SP kernel organisations (generic flat-index kernels in 2D, one plane per
    CTA, no fused coarse tail, the per-step level kernels instead of the fused ones) against the oracle on a ragged grid. A fresh process each: the
    library reads these switches once per process."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _SP_VARIANT.format(root=root)], capture_output=True, text=True,
                       timeout=300, env={**os.environ, **env})
    assert r.returncode == 0 and r.stdout.startswith("ok"), r.stderr[-2000:]


@pytest.mark.parametrize("tma", ["1", "0", "2"])
@pytest.mark.parametrize("shape", [(1, 37, 530), (1, 37, 532), (1, 64, 256), (1, 21, 16)])
def test_sp_staged_rows_parity(tma, shape):
    """The SP level-0 kernels with the rows streamed through a bulk-copy ring (K1
    k_spf_apply_tma for even n_x, the default; with AAC_SPF_TMA=2 also the restriction
    k_spf_restrict_tma and, for n_x % 4 == 0, the prolongation k_spf_prolong_tma: ragged last
    strips, odd n_y, chunk boundaries, a grid smaller than one strip) and the register kernels
    (AAC_SPF_TMA=0) against the oracle. A fresh process each (the switch is read once)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = _SP_VARIANT.format(root=root).replace("shape=(1, 37, 53)", f"shape={shape!r}")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300,
                       env={**os.environ, "AAC_SPF_TMA": tma})
    assert r.returncode == 0 and r.stdout.startswith("ok"), r.stderr[-2000:]


def test_sp_gmres_parity():
    from oracle import saddle
    p = synth.make_problem("saddle", shape=(1, 64, 48))
    s = _solver(p, max_krylov=40)
    x, info = s.gmres("sp", p.k, _dev(p.b, p.ell), rtol=p.rtol, maxit=40)
    w = op.weights(p)
    lev = saddle.hierarchy(w)
    ro = og.fgmres(lambda v: op.apply_allatonce(w, v),
                   lambda v: saddle.sp_apply(w, v, p.ell, p.alpha, p.k, lev), p.b, p.rtol, 40)
    assert info["converged"] == 1 and ro.converged
    assert abs(info["iters"] - ro.iters) <= 1
    assert _rel(x.cpu().numpy(), ro.x) <= 1e-9
    assert info["matvecs_paper_units"] == info["iters"] * (p.ell + 2 * (p.ell - 1) * p.k)
    s.close()


def test_saddle_full_size_gmres_vs_stored_oracle():
    """BASELINE configs[3] (SP, k = 8) at N = 1024^2 vs oracle values stored by
    scripts/make_oracle_golden.py (oracle-only)."""
    g = json.load(open(os.path.join(HERE, "golden", "oracle_saddle.json")))
    p = synth.make_problem("saddle")
    s = _solver(p, max_krylov=40)
    x, info = s.gmres("sp", p.k, _dev(p.b, p.ell), rtol=p.rtol, maxit=40)
    assert abs(info["iters"] - g["iters"]) <= 1 and info["converged"] == 1
    assert info["relres_true"] <= 1.5 * p.rtol
    xs = x.cpu().numpy().ravel()
    idx = np.array(g["sample_idx"])
    ref = np.array(g["sample_x"])
    assert np.linalg.norm(xs[idx] - ref) <= 1e-9 * np.linalg.norm(ref)
    assert np.linalg.norm(xs) == pytest.approx(g["x_norm"], rel=1e-9)
    s.close()


# ---------------------------------------------------------------- NC sweep organisations
# The 2D single-rank NC path runs the wavefront kernel (wave.cuh) by default; depth 4, the
# per-step sweeps (AAC_WAVE_H=0) and small row chunks (AAC_WAVE_LY) must all match the oracle.
WAVE = [
    (dict(shape=(1, 173, 251)), "nc2", 8, "8", "16"),       # 3 strips, 11 chunks, ragged tails
    (dict(shape=(1, 173, 251)), "nc2", 8, "4", "24"),       # two passes per block
    (dict(shape=(1, 173, 251)), "nc2", 8, "0", "0"),        # per-step k_sweep
    (dict(shape=(1, 61, 230)), "nc1", 20, "8", "9"),        # 3 passes, chunks shorter than H+1
    (dict(shape=(1, 61, 230)), "nc1", 20, "4", "0"),
    (dict(shape=(1, 5, 3)), "nc2", 8, "8", "0"),            # grid smaller than the halo
]


@pytest.mark.parametrize("kw,method,k,h,ly", WAVE)
def test_precond_sweep_organisations(monkeypatch, kw, method, k, h, ly):
    monkeypatch.setenv("AAC_WAVE_H", h)
    monkeypatch.setenv("AAC_WAVE_LY", ly)
    p = synth.make_problem("headline", **kw)
    s = _solver(p)
    w = op.weights(p)
    mu = op.gershgorin_max(w)
    al = ch.allocate(p.ell, 1.0, mu, p.alpha, p.ell * k, method, k)
    r = np.random.default_rng(9).standard_normal((p.ell,) + p.shape)
    z = s.precond_apply(method, k, _dev(r, p.ell)).cpu().numpy()
    assert _rel(z, ch.nc_apply(w, r, p.ell, p.alpha, 1.0, mu, al)) <= 1e-12
    x, info = s.gmres(method, k, _dev(p.b, p.ell), rtol=p.rtol, maxit=60)
    ro = _oracle_gmres(p, method, k, 60)
    assert abs(info["iters"] - ro.iters) <= 1
    assert _rel(x.cpu().numpy(), ro.x) <= 1e-9
    s.close()


# The cluster wavefront (k_waver CLU: the strips of a row chunk exchange edge columns through
# distributed shared memory, no x-halo) computes the same points from the same operands as the
# halo kernel: bit-identical, for 2..8 strips per row, ragged last strips and short chunks.
CLUSTER = [
    (dict(shape=(1, 96, 1024)), "nc2", 8, "0"),     # 8 full strips (the headline width)
    (dict(shape=(1, 70, 1000)), "nc2", 8, "16"),    # 8 strips, ragged last strip, 5 chunks
    (dict(shape=(1, 40, 300)), "nc1", 20, "0"),     # 3 strips, two passes (nc1 k=20)
    (dict(shape=(1, 33, 129)), "nc2", 8, "9"),      # 2 strips, the second one column wide
]


@pytest.mark.parametrize("kw,method,k,ly", CLUSTER)
def test_cluster_wavefront_bit_identical(monkeypatch, kw, method, k, ly):
    monkeypatch.setenv("AAC_WAVE_LY", ly)
    p = synth.make_problem("headline", **kw)
    r = np.random.default_rng(11).standard_normal((p.ell,) + p.shape)
    z = {}
    for clu in ("1", "0"):
        monkeypatch.setenv("AAC_WAVE_CLUSTER", clu)
        s = _solver(p)
        z[clu] = s.precond_apply(method, k, _dev(r, p.ell)).cpu().numpy()
        s.close()
    assert np.array_equal(z["1"], z["0"])
    w = op.weights(p)
    mu = op.gershgorin_max(w)
    al = ch.allocate(p.ell, 1.0, mu, p.alpha, p.ell * k, method, k)
    assert _rel(z["1"], ch.nc_apply(w, r, p.ell, p.alpha, 1.0, mu, al)) <= 1e-12


# -------------------------------------------------- traversal direction masks
@pytest.mark.parametrize("kw,method,k", [
    (dict(shape=(1, 150, 301)), "nc2", 8),          # wavefront, ragged strips and chunks
    (dict(shape=(1, 61, 47)), "nc1", 20),           # two passes
])
def test_traversal_direction_masks(monkeypatch, kw, method, k):
    """AAC_REV flips the LOGICAL CTA index of the streaming kernels: calA, the preconditioner
    and a whole GMRES solve are bit-identical for every mask that leaves k_arnoldi alone
    (its persistent CTAs walk their tiles backwards, which reorders their private sums:
    there the iteration count must agree and the solution to rounding), and all match the
    oracle."""
    p = synth.make_problem("headline", **kw)
    rng = np.random.default_rng(17)
    r = rng.standard_normal((p.ell,) + p.shape)
    out = {}
    for m in ("0", "5", "29", "453", "31"):       # 453: the default (5 + the L2 policy bits)
        monkeypatch.setenv("AAC_REV", m)
        s = _solver(p)
        y = s.matvec(_dev(r, p.ell)).cpu().numpy()
        z = s.precond_apply(method, k, _dev(r, p.ell)).cpu().numpy()
        x, info = s.gmres(method, k, _dev(p.b, p.ell), rtol=p.rtol, maxit=60)
        out[m] = (y, z, x.cpu().numpy(), info["iters"])
        s.close()
    for m in ("5", "29", "453"):                       # k_arnoldi forward in 0, 5, 29, 453
        for a, b in zip(out["0"][:3], out[m][:3]):
            assert np.array_equal(a, b)
        assert out[m][3] == out["0"][3]
    assert np.array_equal(out["31"][0], out["0"][0]) and np.array_equal(out["31"][1], out["0"][1])
    assert out["31"][3] == out["0"][3]
    assert _rel(out["31"][2], out["0"][2]) <= 1e-12
    w = op.weights(p)
    mu = op.gershgorin_max(w)
    al = ch.allocate(p.ell, 1.0, mu, p.alpha, p.ell * k, method, k)
    assert _rel(out["5"][0], op.apply_allatonce(w, r)) <= 1e-12
    assert _rel(out["5"][1], ch.nc_apply(w, r, p.ell, p.alpha, 1.0, mu, al)) <= 1e-12


# ---------------------------------------------------------------- full-size 3D (configs[4])
def _sub_weights(w, lo, hi):
    """Face weights of the box [lo, hi) of the full grid (faces inside the box only): the box
    is its own Neumann problem, identical to the full one within its interior."""
    sub = op.Weights.__new__(op.Weights)
    (z0, y0, x0), (z1, y1, x1) = lo, hi
    sub.shape = (z1 - z0, y1 - y0, x1 - x0)
    sub.wx = w.wx[z0:z1, y0:y1, x0:x1 - 1]
    sub.wy = w.wy[z0:z1, y0:y1 - 1, x0:x1]
    sub.wz = w.wz[z0:z1 - 1, y0:y1, x0:x1]
    return sub


def test_3d_full_size_sampled_parity():
    """calA and P_NC1 (k = 10) at 256^3, ell = 12 -- the bench launch configuration -- on sampled
    points. The preconditioner is a polynomial of degree p - 1 = 9 in A per Fourier block, so its
    value at a point depends only on r within 9 cells: the oracle on a 25^3 box around the point
    (the box is a Neumann problem that agrees with the full one inside) gives the exact value."""
    p = synth.make_problem("3d")
    s = _solver(p, max_krylov=16)
    w = op.weights(p)
    mu = op.gershgorin_max(w)
    assert s.mu_max == pytest.approx(mu, rel=1e-14)
    r = np.random.default_rng(13).standard_normal((p.ell,) + p.shape)
    rd = _dev(r, p.ell)
    y = s.matvec(rd).cpu().numpy().reshape((p.ell,) + p.shape)
    z = s.precond_apply("nc1", p.k, rd).cpu().numpy().reshape((p.ell,) + p.shape)
    del rd
    n = p.shape[0]
    R = 12
    al = ch.allocate(p.ell, 1.0, mu, p.alpha, p.ell * p.k, "nc1", p.k)
    for pt in [(0, 0, 0), (5, 130, 255), (128, 127, 129), (255, 3, 77), (200, 255, 0)]:
        lo = tuple(max(0, c - R) for c in pt)
        hi = tuple(min(n, c + R + 1) for c in pt)
        sub = _sub_weights(w, lo, hi)
        sl = (slice(None),) + tuple(slice(a, b) for a, b in zip(lo, hi))
        ctr = (slice(None),) + tuple(c - a for c, a in zip(pt, lo))
        yo = op.apply_allatonce(sub, r[sl]).reshape((p.ell,) + sub.shape)[ctr]
        zo = ch.nc_apply(sub, r[sl], p.ell, p.alpha, 1.0, mu, al).reshape((p.ell,) + sub.shape)[ctr]
        gi = (slice(None),) + pt
        assert _rel(y[gi], yo) <= 1e-12, pt
        assert _rel(z[gi], zo) <= 1e-12, pt
    s.close()


def test_3d_full_size_gmres_properties():
    """configs[4] solve at full size: converged to rtol on the TRUE residual, iteration count in
    the band the survey's 64^3 proxy and the 1-GPU bench show (11)."""
    p = synth.make_problem("3d")
    s = _solver(p, max_krylov=16)
    x, info = s.gmres("nc1", p.k, _dev(p.b, p.ell), rtol=p.rtol, maxit=16)
    assert info["converged"] == 1 and 9 <= info["iters"] <= 13
    assert info["relres_true"] <= 1.5 * p.rtol
    s.close()
