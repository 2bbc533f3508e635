"""Pins for oracle/varying.py (CPU only).

The paper prints no numbers for varying blocks, so the pins are the definitions: the block
system against an assembly of its sparse blocks, the sequential recurrence against a dense
solve, the average operator against the average of the operators, the equal-block limit
against the constant-block operator, and GMRES with P_alpha(A_hat) reaching x*.
"""
import numpy as np
import pytest
import scipy.sparse as sp

import synth
from oracle import chebyshev as ch
from oracle import gmres as og
from oracle import operator as op
from oracle import varying as va


def _ws(shape=(1, 6, 7), ell=4, drift=0.8, name="headline"):
    p = synth.make_varying_problem(name, shape=shape, ell=ell, drift=drift)
    return p, va.block_weights(p)


def _block_matrix(ws):
    ell = len(ws)
    N = ws[0].N
    D = sp.block_diag([op.sparse_A(w) for w in ws]).tocsr()
    S = sp.kron(sp.eye(ell, k=-1), sp.eye(N))
    return (D - S).toarray()


@pytest.mark.parametrize("shape,ell", [((1, 6, 7), 4), ((3, 4, 5), 6)])
def test_block_apply_equals_assembly(shape, ell):
    p, ws = _ws(shape, ell, name="3d" if shape[0] > 1 else "headline")
    x = np.random.default_rng(2).standard_normal((ell,) + shape)
    y = va.apply_allatonce_var(ws, x)
    assert np.allclose(y.ravel(), _block_matrix(ws) @ x.ravel(), rtol=1e-13, atol=1e-12)
    v = np.zeros_like(x)
    v[0] = x[0]
    yv = va.apply_allatonce_var(ws, v)                       # (v, 0, ...) -> (A_1 v, -v, 0, ...)
    assert np.allclose(yv[0], op.apply_A(ws[0], x[0])) and np.allclose(yv[1], -x[0])
    assert not np.any(yv[2:])


def test_blocks_really_vary_and_drift_zero_is_constant():
    p, ws = _ws(drift=0.8)
    assert np.max(np.abs(ws[0].wx - ws[-1].wx)) > 0.05 * np.max(ws[0].wx)
    p0, ws0 = _ws(drift=0.0)
    x = np.random.default_rng(3).standard_normal((p0.ell,) + p0.shape)
    assert np.array_equal(va.apply_allatonce_var(ws0, x), op.apply_allatonce(ws0[0], x))


def test_recurrence_equals_dense_solve():
    p, ws = _ws()
    b = np.random.default_rng(4).standard_normal((p.ell,) + p.shape)
    x = va.solve_recurrence_var(ws, b)
    xd = np.linalg.solve(_block_matrix(ws), b.ravel())
    assert np.allclose(x.ravel(), xd, rtol=1e-12, atol=1e-12)


def test_mean_weights_is_mean_operator():
    p, ws = _ws()
    wh = va.mean_weights(ws)
    u = np.random.default_rng(5).standard_normal(p.shape)
    mean_op = np.mean([op.apply_A(w, u) for w in ws], axis=0)
    assert np.allclose(op.apply_A(wh, u), mean_op, rtol=1e-14, atol=1e-13)


def test_gmres_with_mean_block_preconditioner_reaches_x_star():
    p, ws = _ws(shape=(1, 12, 10), ell=10)
    wh = va.mean_weights(ws)
    mu = op.gershgorin_max(wh)
    al = ch.allocate(p.ell, 1.0, mu, p.alpha, p.ell * 8, "nc2")
    res = og.fgmres(lambda v: va.apply_allatonce_var(ws, v),
                    lambda r: ch.nc_apply(wh, r, p.ell, p.alpha, 1.0, mu, al), p.b, 1e-10, 60)
    xs = va.solve_recurrence_var(ws, p.b)
    assert res.converged
    assert np.linalg.norm(res.x - xs) <= 1e-7 * np.linalg.norm(xs)
