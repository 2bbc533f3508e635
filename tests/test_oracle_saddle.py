"""Pins for oracle/saddle.py (CPU only).

Pinned against: the dense 2N saddle assembly and the complex solve it encodes
(Eq. eq:saddlesystem); the eigenvalue interval of
Thm with exact P_D; scipy.sparse.linalg.minres / cg iterates
(library routines) for the same k; V-cycle symmetry, positive definiteness and
contraction; Galerkin coarse operators keep the face
form (coarse face = sum of fine faces crossing it, mass = child count); P_SP -> the
exact P_alpha^{-1} as k grows.
"""
import math

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from oracle import circulant as circ
from oracle import operator as op
from oracle import saddle


def _w(shape=(1, 6, 7), seed=0, c=None):
    rng = np.random.default_rng(seed)
    nz, ny, nx = shape
    return op.Weights(shape, 0.6 / nx ** 2 if c is None else c,
                      np.exp(0.3 * rng.standard_normal((nz, ny, nx - 1))),
                      np.exp(0.3 * rng.standard_normal((nz, ny - 1, nx))),
                      np.exp(0.3 * rng.standard_normal((nz - 1, ny, nx))))


LAMS = [0.3 + 0.5j, -0.6 + 0.2j, 0.9 + 0.05j]


@pytest.mark.parametrize("lam", LAMS)
def test_saddle_encodes_complex_solve(lam):
    w = _w()
    A = op.dense_A(w)
    rng = np.random.default_rng(1)
    b = rng.standard_normal(w.N) + 1j * rng.standard_normal(w.N)
    S = saddle.saddle_dense(A, lam)
    uv = np.linalg.solve(S, np.concatenate([-b.imag, b.real]))
    x = uv[:w.N] - 1j * uv[w.N:]
    assert np.linalg.norm((A - lam * np.eye(w.N)) @ x - b) <= 1e-12 * np.linalg.norm(b)
    t = rng.standard_normal(2 * w.N)
    assert np.allclose(saddle.saddle_apply(w, lam, t), S @ t, atol=1e-13)
    assert np.allclose(S, S.T)


@pytest.mark.parametrize("lam", LAMS)
def test_theorem_41_interval(lam):
    A = op.dense_A(_w((1, 4, 5)))
    N = A.shape[0]
    S = saddle.saddle_dense(A, lam)
    PD = np.kron(np.eye(2), A + (lam.imag - lam.real) * np.eye(N))
    ev = np.linalg.eigvals(np.linalg.solve(PD, S))
    assert np.abs(ev.imag).max() < 1e-10
    a = np.abs(ev.real)
    assert a.min() >= 1 / math.sqrt(2) - 1e-10 and a.max() <= 1 + 1e-10


@pytest.mark.parametrize("lam", LAMS[:2])
@pytest.mark.parametrize("k", [1, 3, 8])
def test_minres_matches_scipy(lam, k):
    w = _w()
    A = op.dense_A(w)
    N = w.N
    S = saddle.saddle_dense(A, lam)
    Minv = np.linalg.inv(np.kron(np.eye(2), A + (lam.imag - lam.real) * np.eye(N)) + 0.3 * np.eye(2 * N))
    b = np.random.default_rng(2).standard_normal(2 * N)
    x = saddle.minres(lambda v: S @ v, lambda v: Minv @ v, b, k)
    xs, _ = spla.minres(S, b, rtol=0.0, maxiter=k, M=Minv)
    assert np.linalg.norm(x - xs) <= 1e-10 * np.linalg.norm(xs)
    # preconditioned residual norm non-increasing in k
    if k > 1:
        xm = saddle.minres(lambda v: S @ v, lambda v: Minv @ v, b, k - 1)
        rn = lambda y: float((b - S @ y) @ (Minv @ (b - S @ y)))
        assert rn(x) <= rn(xm) * (1 + 1e-12)


@pytest.mark.parametrize("k", [1, 4, 8])
def test_pcg_matches_scipy(k):
    w = _w()
    A = op.dense_A(w) + 0.4 * np.eye(w.N)
    M = np.linalg.inv(np.diag(np.diag(A)))
    b = np.random.default_rng(3).standard_normal(w.N)
    x = saddle.pcg(lambda v: A @ v, lambda v: M @ v, b, k)
    xs, _ = spla.cg(A, b, rtol=0.0, atol=0.0, maxiter=k, M=M)
    assert np.linalg.norm(x - xs) <= 1e-10 * np.linalg.norm(xs)


@pytest.mark.parametrize("shape", [(1, 1, 40), (1, 19, 22), (1, 24, 24), (11, 10, 9)])
@pytest.mark.parametrize("s", [0.4, -0.39])
def test_vcycle_symmetric_pd_contracting(shape, s):
    w = _w(shape, c=2.0 / shape[2] ** 2 * 3)
    lev = saddle.hierarchy(w)
    assert len(lev) >= 2 and max(lev[-1].shape) <= saddle.COARSEST_MAX_AXIS
    N = w.N
    Bm = np.column_stack([saddle.vcycle(lev, s, e) for e in np.eye(N)])
    assert np.abs(Bm - Bm.T).max() <= 1e-12 * np.abs(Bm).max()
    assert np.linalg.eigvalsh(0.5 * (Bm + Bm.T)).min() > 0
    A = op.dense_A(w) + s * np.eye(N)
    rho = np.abs(np.linalg.eigvals(np.eye(N) - Bm @ A)).max()
    assert rho < 0.9


def test_galerkin_coarse_keeps_face_form():
    """P^T (A + sI) P = s'*diag(cnt) + graph Laplacian whose coarse face weight is the sum
    of the fine faces between the two aggregates (the GPU builds coarse levels this way)."""
    w = _w((1, 7, 9))
    lev = saddle.hierarchy(w)
    c1 = lev[1]
    A0 = c1.A0.toarray()
    cnt = c1.cnt
    L = A0 - np.diag(cnt)                           # graph Laplacian part
    assert np.allclose(L.sum(axis=1), 0, atol=1e-12)
    assert (np.diag(L) >= 0).all() and (L - np.diag(np.diag(L)) <= 1e-15).all()
    # coarse x-face between aggregates (I, J) and (I+1, J) = sum of fine x-faces crossing it
    cy, cx = c1.shape[1], c1.shape[2]
    for J in range(cy):
        for I in range(cx - 1):
            fine = sum(w.wx[0, j, 2 * I + 1] for j in (2 * J, 2 * J + 1) if j < 7)
            assert -L[J * cx + I, J * cx + I + 1] == pytest.approx(fine, rel=1e-14)
    assert sorted(set(cnt.tolist())) == [1.0, 2.0, 4.0]


def test_sp_converges_to_exact():
    w = _w((1, 10, 12), seed=4)
    ell, alpha = 6, 1e-2
    r = np.random.default_rng(5).standard_normal((ell,) + w.shape)
    z = circ.exact_apply(w, r, ell, alpha)
    lev = saddle.hierarchy(w)
    errs = [np.linalg.norm(saddle.sp_apply(w, r, ell, alpha, k, lev) - z) / np.linalg.norm(z)
            for k in (2, 6, 40)]
    assert errs[0] > errs[1] > errs[2] and errs[2] < 1e-8
