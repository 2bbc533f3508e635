"""Pins for oracle/operator.py (CPU only).

Pinned against: an independent sparse assembly A = I + G^T W G; the Neumann null
mode A.1 = 1; symmetry/positive definiteness; the kappa = 1 closed-form DCT-II
eigenpairs; the block structure of Eq. (eq:A); the Kronecker
form; the dense direct solve of calA x = b.
"""
import math

import numpy as np
import pytest

import synth
from oracle import operator as op

SHAPES = [(1, 1, 9), (1, 5, 7), (1, 6, 4), (3, 4, 5)]


def _w(shape, seed=0, c=None):
    rng = np.random.default_rng(seed)
    nz, ny, nx = shape
    kx = np.exp(rng.standard_normal((nz, ny, nx - 1)) * 0.3)
    ky = np.exp(rng.standard_normal((nz, ny - 1, nx)) * 0.3)
    kz = np.exp(rng.standard_normal((nz - 1, ny, nx)) * 0.3)
    return op.Weights(shape, 0.7 / (nx * nx) if c is None else c, kx, ky, kz)


@pytest.mark.parametrize("shape", SHAPES)
def test_matrix_free_equals_graph_laplacian_assembly(shape):
    w = _w(shape)
    A = op.dense_A(w)
    u = np.random.default_rng(1).standard_normal(w.N)
    assert np.allclose(op.apply_A(w, u).ravel(), A @ u, rtol=1e-14, atol=1e-13)
    # explicit stencil entries: brute-force per cell from the face list
    nz, ny, nx = shape
    Ab = np.eye(w.N)
    idx = np.arange(w.N).reshape(shape)
    for (k, j, i), P in np.ndenumerate(idx):
        for (dk, dj, di, wf) in ((0, 0, 1, w.wx[k, j, i] if i < nx - 1 else 0),
                                 (0, 0, -1, w.wx[k, j, i - 1] if i > 0 else 0),
                                 (0, 1, 0, w.wy[k, j, i] if j < ny - 1 else 0),
                                 (0, -1, 0, w.wy[k, j - 1, i] if j > 0 else 0),
                                 (1, 0, 0, w.wz[k, j, i] if k < nz - 1 else 0),
                                 (-1, 0, 0, w.wz[k - 1, j, i] if k > 0 else 0)):
            if wf:
                Ab[P, P] += wf
                Ab[P, idx[k + dk, j + dj, i + di]] -= wf
    assert np.allclose(Ab, A, rtol=1e-14, atol=1e-14)


@pytest.mark.parametrize("shape", SHAPES)
def test_neumann_constant_mode_and_spd(shape):
    w = _w(shape)
    A = op.dense_A(w)
    one = np.ones(w.N)
    assert np.allclose(op.apply_A(w, one).ravel(), one, atol=1e-13)   # A.1 = 1 -> mu_min = 1
    assert np.allclose(A, A.T, atol=0)
    ev = np.linalg.eigvalsh(A)
    assert ev.min() == pytest.approx(1.0, abs=1e-12)
    assert ev.max() <= op.gershgorin_max(w) * (1 + 1e-14)


@pytest.mark.parametrize("shape", SHAPES)
def test_gershgorin_equals_dense_row_sums(shape):
    """gershgorin_max is THE Gershgorin bound max_i (a_ii + sum_{j != i} |a_ij|) of the
    brute-force per-cell assembly above (reading R5), not merely some upper bound."""
    w = _w(shape)
    nz, ny, nx = shape
    idx = np.arange(w.N).reshape(shape)
    Ab = np.eye(w.N)
    for (k, j, i), P in np.ndenumerate(idx):
        for (dk, dj, di, wf) in ((0, 0, 1, w.wx[k, j, i] if i < nx - 1 else 0),
                                 (0, 0, -1, w.wx[k, j, i - 1] if i > 0 else 0),
                                 (0, 1, 0, w.wy[k, j, i] if j < ny - 1 else 0),
                                 (0, -1, 0, w.wy[k, j - 1, i] if j > 0 else 0),
                                 (1, 0, 0, w.wz[k, j, i] if k < nz - 1 else 0),
                                 (-1, 0, 0, w.wz[k - 1, j, i] if k > 0 else 0)):
            if wf:
                Ab[P, P] += wf
                Ab[P, idx[k + dk, j + dj, i + di]] -= wf
    dense = max(Ab[i, i] + np.sum(np.abs(Ab[i])) - abs(Ab[i, i]) for i in range(w.N))
    assert op.gershgorin_max(w) == pytest.approx(dense, rel=1e-15)


@pytest.mark.parametrize("name,printed", [("1d", 36.61), ("2d256", 50.81), ("headline", 32.14)])
def test_gershgorin_survey_values(name, printed):
    """mu_max of the seeded BASELINE configs as printed by the survey's independent numpy
    prototype ("Est. mu_max", seed 0), to the printed 4 digits."""
    w = op.weights(synth.make_problem(name))
    assert round(op.gershgorin_max(w), 2) == printed


@pytest.mark.parametrize("shape", [(1, 1, 16), (1, 8, 12), (4, 6, 5)])
def test_kappa_one_closed_form_dct(shape):
    """kappa = 1: A cos-modes prod_a cos(pi m_a (i_a + 1/2)/n_a) have eigenvalue
    1 + sum_a 4 w_a sin^2(pi m_a / (2 n_a)) (DCT-II diagonalises the Neumann Laplacian)."""
    nz, ny, nx = shape
    c = 0.37 / (nx * nx)
    w = op.Weights(shape, c, np.ones((nz, ny, nx - 1)), np.ones((nz, ny - 1, nx)),
                   np.ones((nz - 1, ny, nx)))
    rng = np.random.default_rng(2)
    for _ in range(6):
        m = [rng.integers(0, n) for n in shape]
        K, J, I = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
        v = (np.cos(math.pi * m[0] * (K + 0.5) / nz) * np.cos(math.pi * m[1] * (J + 0.5) / ny)
             * np.cos(math.pi * m[2] * (I + 0.5) / nx))
        lam = 1.0
        for ma, na in zip(m, shape):
            if na > 1:
                lam += 4.0 * c * na * na * math.sin(math.pi * ma / (2 * na)) ** 2
        assert np.allclose(op.apply_A(w, v), lam * v, atol=1e-12 * lam)


def test_c_zero_is_identity():
    w = _w((1, 5, 6), c=0.0)
    u = np.random.default_rng(3).standard_normal(w.shape)
    assert np.array_equal(op.apply_A(w, u), u)
    assert op.gershgorin_max(w) == 1.0


def test_allatonce_block_structure():
    """(v, 0, ..., 0) -> (A v, -v, 0, ..., 0)."""
    w = _w((1, 5, 7))
    ell = 6
    v = np.random.default_rng(4).standard_normal(w.shape)
    x = np.zeros((ell,) + w.shape)
    x[0] = v
    y = op.apply_allatonce(w, x)
    assert np.allclose(y[0], op.apply_A(w, v))
    assert np.array_equal(y[1], -v)
    assert not y[2:].any()


@pytest.mark.parametrize("ell", [2, 4, 6])
def test_allatonce_equals_kronecker(ell):
    w = _w((1, 4, 3))
    A = op.dense_A(w)
    K = op.dense_allatonce(A, ell)
    x = np.random.default_rng(5).standard_normal((ell,) + w.shape)
    assert np.allclose(op.apply_allatonce(w, x).ravel(), K @ x.ravel(), atol=1e-13)
    # c = 0: unit lower block bidiagonal
    w0 = _w((1, 4, 3), c=0.0)
    K0 = op.dense_allatonce(op.dense_A(w0), ell)
    assert np.array_equal(K0, np.eye(ell * w0.N) - np.eye(ell * w0.N, k=-w0.N))


def test_recurrence_equals_dense_solve():
    w = _w((1, 5, 4))
    ell = 6
    b = np.random.default_rng(6).standard_normal((ell,) + w.shape)
    x = op.solve_recurrence(w, b)
    xd = np.linalg.solve(op.dense_allatonce(op.dense_A(w), ell), b.ravel())
    assert np.allclose(x.ravel(), xd, rtol=1e-13, atol=1e-13)


def test_input_generator_recipe():
    """Synth inputs: kappa > 0, b = (b_1, 0, ...), the 256^2 and 1024^2 fields are the
    same function (same draws), anisotropy 0.25 on y faces of the headline."""
    p = synth.make_problem("2d256", n=16)
    q = synth.make_problem("headline", n=16)
    assert (p.kx > 0).all() and (p.ky > 0).all()
    assert not p.b[1:].any() and p.b[0].any()
    assert np.allclose(q.kx, p.kx) and np.allclose(q.ky, 0.25 * p.ky)
    assert p.c == pytest.approx((10.0 / 16) ** 2 / 20.0)
    d = synth.make_problem("1d")
    w = op.weights(d)
    assert w.wx.shape == (1, 1, 127) and d.ell == 4
    assert np.allclose(w.wx / d.kx, 8.0)          # c/h^2 = (L/h)^2/(2 ell) = 64/8
