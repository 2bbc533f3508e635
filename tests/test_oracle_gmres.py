"""Pins for oracle/gmres.py (CPU only).

Pinned against: scipy.sparse.linalg.gmres iterates (library routine, unpreconditioned,
same Krylov space -> same minimiser); the exact solution by the recurrence; the
closed-form special case c = 0 (A = I): P_alpha^{-1} calA has eigenvalues {1, 1/(1-alpha)}
(Thm thm:evals) so GMRES converges in exactly 1 iteration for
b = (b_1, 0, ..., 0) (an eigenvector: P_alpha 1 = (1-alpha) e_1 per point) and in
exactly 2 for a generic right-hand side.
"""
import numpy as np
import pytest
import scipy.sparse.linalg as spla

import synth
from oracle import chebyshev as ch
from oracle import circulant as circ
from oracle import gmres
from oracle import operator as op


def test_matches_scipy_gmres_unpreconditioned():
    p = synth.make_problem("2d256", n=8, ell=4)
    w = op.weights(p)
    K = op.dense_allatonce(op.dense_A(w), p.ell)
    b = p.b.reshape(-1)
    for m in (1, 3, 6):
        res = gmres.fgmres(lambda x: op.apply_allatonce(w, x), lambda v: v, p.b, rtol=0.0, maxit=m)
        x_sp, _ = spla.gmres(K, b, rtol=0.0, atol=0.0, restart=m, maxiter=1)
        assert res.iters == m
        assert np.linalg.norm(res.x.ravel() - x_sp) <= 1e-10 * np.linalg.norm(x_sp)
        # Arnoldi residual estimate equals the true residual
        tr = np.linalg.norm(b - K @ res.x.ravel()) / np.linalg.norm(b)
        assert res.relres_est == pytest.approx(tr, rel=1e-8)


@pytest.mark.parametrize("rhs,expect", [("b1", 1), ("all", 2)])
def test_c_zero_exact_counts(rhs, expect):
    p = synth.make_problem("headline", n=16, c=0.0, rhs=rhs)
    w = op.weights(p)
    mu = op.gershgorin_max(w)
    assert mu == 1.0
    res = gmres.fgmres(lambda x: op.apply_allatonce(w, x),
                       lambda r: ch.nc_apply(w, r, p.ell, p.alpha, 1.0, mu, [1] * p.ell),
                       p.b, rtol=1e-10, maxit=20)
    assert res.iters == expect and res.converged


def test_solution_vs_recurrence_1d_config():
    p = synth.make_problem("1d")
    w = op.weights(p)
    mu = op.gershgorin_max(w)
    al = ch.allocate(p.ell, 1.0, mu, p.alpha, p.ell * p.k, "nc1", p.k)
    res = gmres.fgmres(lambda x: op.apply_allatonce(w, x),
                       lambda r: ch.nc_apply(w, r, p.ell, p.alpha, 1.0, mu, al), p.b, 1e-10, 200)
    xs = op.solve_recurrence(w, p.b)
    assert res.converged
    tr = np.linalg.norm(p.b - op.apply_allatonce(w, res.x)) / np.linalg.norm(p.b)
    assert tr <= 1e-10 * 1.01
    # ||x - x*|| <= kappa(calA) * relres * ||x*||, kappa(calA) <= ell (mu_max + 1)
    assert np.linalg.norm(res.x - xs) <= p.ell * (mu + 1) * 1e-10 * np.linalg.norm(xs)


def test_exact_preconditioner_small_alpha_converges_fast():
    """With exact P_alpha and tiny alpha (eigenvalues clustered at 1, Cor. 2.4) GMRES needs
    very few iterations (1 outer CI iteration for alpha <= 1e-5)."""
    p = synth.make_problem("2d256", n=8, alpha=1e-6)
    w = op.weights(p)
    res = gmres.fgmres(lambda x: op.apply_allatonce(w, x),
                       lambda r: circ.exact_apply(w, r, p.ell, p.alpha), p.b, 1e-10, 20)
    assert res.converged and res.iters <= 3
