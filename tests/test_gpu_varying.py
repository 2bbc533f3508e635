"""Varying diagonal blocks A_1..A_ell on the GPU vs the oracle
(oracle/varying.py): the block operator apply to 1e-12, the mean-block preconditioner to 1e-12,
GMRES counts +-1 and solutions 1e-9, and the refusal of the outer CI the paper rules out."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import synth  # noqa: E402
from oracle import chebyshev as ch  # noqa: E402
from oracle import gmres as og  # noqa: E402
from oracle import operator as op  # noqa: E402
from oracle import varying as va  # noqa: E402


def _dev(a, ell):
    return torch.from_numpy(np.ascontiguousarray(a).reshape(ell, -1)).cuda()


def _rel(a, b):
    a, b = np.asarray(a).ravel(), np.asarray(b).ravel()
    return np.linalg.norm(a - b) / np.linalg.norm(b)


CASES = [("headline", dict(shape=(1, 130, 67))), ("headline", dict(shape=(1, 64, 64), ell=4)),
         ("3d", dict(shape=(9, 13, 11))), ("1d", {})]


@pytest.mark.parametrize("name,kw", CASES)
def test_varying_apply_and_precond_parity(name, kw):
    from paper_2506_03947_b200 import from_problem
    p = synth.make_varying_problem(name, drift=0.8, **kw)
    s = from_problem(p, max_krylov=8)
    ws = va.block_weights(p)
    wh = va.mean_weights(ws)
    assert s.mu_max == pytest.approx(op.gershgorin_max(wh), rel=1e-14)
    x = np.random.default_rng(7).standard_normal((p.ell,) + p.shape)
    assert _rel(s.matvec(_dev(x, p.ell)).cpu().numpy(), va.apply_allatonce_var(ws, x)) <= 1e-12
    al = ch.allocate(p.ell, 1.0, op.gershgorin_max(wh), p.alpha, p.ell * 6, "nc2")
    z = s.precond_apply("nc2", 6, _dev(x, p.ell)).cpu().numpy()
    assert _rel(z, ch.nc_apply(wh, x, p.ell, p.alpha, 1.0, op.gershgorin_max(wh), al)) <= 1e-12
    s.close()


@pytest.mark.parametrize("name,kw,method,k", [("headline", dict(shape=(1, 100, 73)), "nc2", 8),
                                              ("headline", dict(n=256), "nc1", 8),
                                              ("3d", dict(shape=(16, 16, 16)), "nc1", 10)])
def test_varying_gmres_parity(name, kw, method, k):
    from paper_2506_03947_b200 import from_problem
    p = synth.make_varying_problem(name, drift=0.8, **kw)
    s = from_problem(p, max_krylov=60)
    ws = va.block_weights(p)
    wh = va.mean_weights(ws)
    mu = op.gershgorin_max(wh)
    al = ch.allocate(p.ell, 1.0, mu, p.alpha, p.ell * k, method, k)
    ro = og.fgmres(lambda v: va.apply_allatonce_var(ws, v),
                   lambda r: ch.nc_apply(wh, r, p.ell, p.alpha, 1.0, mu, al), p.b, p.rtol, 60)
    x, info = s.gmres(method, k, _dev(p.b, p.ell), rtol=p.rtol, maxit=60)
    assert ro.converged and info["converged"] == 1
    assert abs(info["iters"] - ro.iters) <= 1
    assert _rel(x.cpu().numpy(), ro.x) <= 1e-9
    assert info["relres_true"] <= 1.5 * p.rtol
    s.close()


def test_varying_refuses_outer_ci():
    from paper_2506_03947_b200 import AacError, from_problem
    p = synth.make_varying_problem("headline", shape=(1, 16, 16))
    s = from_problem(p, max_krylov=8)
    with pytest.raises(AacError, match="PAPER.md:991"):
        s.ci("nc2", 4, _dev(p.b, p.ell), lmin=1.0, lmax=2.0)
    s.close()


# ---------------------------------------------------------------- mixed precision (N4)
@pytest.mark.parametrize("method,k,kw", [("nc2", 8, dict(shape=(1, 130, 67))), ("nc1", 8, dict(n=256)),
                                         ("nc2", 8, dict(shape=(1, 61, 230), ell=16, alpha=0.3))])
def test_mixed_precision_apply_and_gmres(method, k, kw):
    """AAC_F32 ("nc2-f32"): the Chebyshev recurrence in fp32 on the GPU vs the oracle's fp32
    variant (oracle/chebyshev.py nc_apply_f32) -- both fp32, different rounding orders, so to fp32
    accuracy (1e-6 x kappa(Gamma)), not bit for bit; FGMRES (fp64) with it converges to rtol and
    its solution matches the fp64 oracle solve within the forward-error bound of rtol."""
    from oracle import circulant as circ
    from paper_2506_03947_b200 import from_problem
    p = synth.make_problem("headline", **kw)
    s = from_problem(p, max_krylov=60)
    w = op.weights(p)
    mu = op.gershgorin_max(w)
    al = ch.allocate(p.ell, 1.0, mu, p.alpha, p.ell * k, method, k)
    r = np.random.default_rng(12).standard_normal((p.ell,) + p.shape)
    z = s.precond_apply(method + "-f32", k, _dev(r, p.ell)).cpu().numpy()
    kg = circ.gamma_condition(p.ell, p.alpha)
    assert _rel(z, ch.nc_apply_f32(w, r, p.ell, p.alpha, 1.0, mu, al)) <= 1e-6 * kg
    z64 = ch.nc_apply(w, r, p.ell, p.alpha, 1.0, mu, al)
    assert 1e-10 < _rel(z, z64) <= 1e-6 * kg                  # really fp32, and close to fp64
    x, info = s.gmres(method + "-f32", k, _dev(p.b, p.ell), rtol=p.rtol, maxit=60)
    ro = og.fgmres(lambda v: op.apply_allatonce(w, v), lambda v: ch.nc_apply(w, v, p.ell, p.alpha, 1.0, mu, al),
                   p.b, p.rtol, 60)
    assert info["converged"] == 1 and info["relres_true"] <= 1.5 * p.rtol
    assert ro.iters - 1 <= info["iters"] <= ro.iters + 2
    assert _rel(x.cpu().numpy(), ro.x) <= p.ell * (mu + 1) * p.rtol
    s.close()


def test_mixed_precision_refused_off_the_wavefront():
    from paper_2506_03947_b200 import AacError, from_problem
    p = synth.make_problem("3d", shape=(9, 13, 11))
    s = from_problem(p, max_krylov=8)
    with pytest.raises(AacError, match="AAC_F32"):
        s.precond_apply("nc1-f32", 4, _dev(np.ones((p.ell, p.N)), p.ell))
    with pytest.raises(AacError, match="AAC_F32"):
        s.precond_apply("sp-f32" if False else 3 | 16, 4, _dev(np.ones((p.ell, p.N)), p.ell))
    s.close()
