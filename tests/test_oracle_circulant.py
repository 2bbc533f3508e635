"""Pins for oracle/circulant.py (CPU only).

Pinned against: the eigenvalues of C_alpha (dense eig; the paper's printed
lambda_2, lambda_3); the dense Kronecker P_alpha of Eq. (eq:exactPBE); the SMW
form of Lemma lemma:Zalpha; Theorem thm:evals and Corollary cor:extremeevals
(dense spectra); kappa(U^* Gamma) closed form vs dense SVD.
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import circulant as circ
from oracle import operator as op

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_scalars.json")))


def _w(shape=(1, 3, 4), seed=0, c=None):
    rng = np.random.default_rng(seed)
    nz, ny, nx = shape
    return op.Weights(shape, 0.5 / nx ** 2 if c is None else c,
                      np.exp(0.3 * rng.standard_normal((nz, ny, nx - 1))),
                      np.exp(0.3 * rng.standard_normal((nz, ny - 1, nx))),
                      np.exp(0.3 * rng.standard_normal((nz - 1, ny, nx))))


@pytest.mark.parametrize("ell,alpha", [(4, 0.3), (6, 1e-2), (10, 1.0), (10, 1e-4), (12, 1e-4)])
def test_C_alpha_eigenvalues(ell, alpha):
    ev = np.linalg.eigvals(circ.C_alpha(ell, alpha))
    lam = circ.shifts(ell, alpha)
    # same multiset as alpha^{1/ell} e^{2 pi i k/ell}
    d = np.abs(ev[:, None] - lam[None, :])
    assert d.min(axis=1).max() < 1e-12 and d.min(axis=0).max() < 1e-12
    assert np.prod(lam) == pytest.approx((-1) ** (ell + 1) * alpha, rel=1e-12)
    assert np.allclose(np.abs(lam), alpha ** (1.0 / ell))


def test_printed_roots_ell10():
    g = GOLD["roots_ell10_alpha1"]
    lam = circ.paper_roots(10, 1.0)
    assert round(lam[1].real, 4) == g["lambda2"][0] and round(lam[1].imag, 4) == g["lambda2"][1]
    assert round(lam[2].real, 4) == g["lambda3"][0] and round(lam[2].imag, 4) == g["lambda3"][1]
    # our Lambda_k is the conjugate labelling (reading R6): same real parts
    assert np.allclose(circ.shifts(10, 1.0)[1], np.conj(lam[1]))


def _F(ell):
    j = np.arange(ell)
    return np.exp(-2j * np.pi * np.outer(j, j) / ell) / math.sqrt(ell)


@pytest.mark.parametrize("ell,alpha", [(4, 0.3), (6, 0.01), (10, 1e-4)])
def test_corrected_factorisation(ell, alpha):
    """C_alpha = Gamma^{-1} F^* Lambda F Gamma with the corrected pairing."""
    F = _F(ell)
    G = np.diag(circ.gammas(ell, alpha))
    Cf = np.linalg.inv(G) @ F.conj().T @ np.diag(circ.shifts(ell, alpha)) @ F @ G
    # rounding is amplified by kappa(Gamma) = alpha^{-(ell-1)/ell} (Fig. 2 right)
    assert np.abs(Cf - circ.C_alpha(ell, alpha)).max() < 1e-15 * 10 * circ.gamma_condition(ell, alpha)


def test_printed_pairing_fails():
    """PAPER.md:240-246 literally (U columns e^{+2pi i (m-1)(j-1)/ell}, lambda_j =
    alpha^{1/ell} e^{+2pi i (j-1)/ell}) does not give C_alpha -> reading R6."""
    ell, alpha = 4, 0.3
    U = _F(ell).conj()                  # U_j = ell^{-1/2}(e^{2 pi i (m-1)(j-1)/ell})_m
    G = np.diag(circ.gammas(ell, alpha))
    Cp = np.linalg.inv(G) @ U @ np.diag(circ.paper_roots(ell, alpha)) @ U.conj().T @ G
    assert np.abs(Cp - circ.C_alpha(ell, alpha)).max() > 1.0


def test_forward_inverse():
    ell, alpha = 6, 0.05
    r = np.random.default_rng(1).standard_normal((ell, 1, 3, 4))
    assert np.allclose(circ.inverse(circ.forward(r, ell, alpha), ell, alpha), r, atol=1e-13)
    v = np.random.default_rng(2).standard_normal((1, 3, 4))
    c = np.broadcast_to(v, (ell, 1, 3, 4))
    h = circ.forward(c, ell, 1.0)        # alpha = 1, constant blocks -> sqrt(ell) v in block 0
    assert np.allclose(h[0], math.sqrt(ell) * v) and np.abs(h[1:]).max() < 1e-14


@pytest.mark.parametrize("ell,alpha", [(4, 0.3), (6, 1e-2), (10, 1e-4)])
def test_exact_apply_equals_dense_inverse_and_smw(ell, alpha):
    w = _w()
    A = op.dense_A(w)
    P = circ.dense_P_alpha(A, ell, alpha)
    r = np.random.default_rng(3).standard_normal((ell,) + w.shape)
    z = circ.exact_apply(w, r, ell, alpha)
    zd = np.linalg.solve(P, r.ravel())
    assert np.linalg.norm(z.ravel() - zd) <= 1e-12 * np.linalg.norm(zd) * circ.gamma_condition(ell, alpha)
    S = circ.smw_inverse(A, ell, alpha)
    assert np.allclose(S @ r.ravel(), zd, rtol=1e-10, atol=1e-12)
    # P_alpha = calA - alpha E_1 E_ell^T
    N = w.N
    K = op.dense_allatonce(A, ell)
    K[:N, -N:] -= alpha * np.eye(N)
    assert np.array_equal(K, P)


@pytest.mark.parametrize("ell,alpha", [(4, 1e-2), (6, 0.5), (4, 0.9)])
def test_theorem_evals_and_corollary(ell, alpha):
    """spec(P^{-1} calA) = {1 x (ell-1)N} U {mu^ell/(mu^ell - alpha)}; max = 1/(1-alpha)
    since mu_min = 1 under Neumann."""
    w = _w((1, 3, 3))
    A = op.dense_A(w)
    N = w.N
    M = np.linalg.solve(circ.dense_P_alpha(A, ell, alpha), op.dense_allatonce(A, ell))
    ev = np.sort_complex(np.linalg.eigvals(M))
    mu = np.linalg.eigvalsh(A)
    expect = np.sort_complex(np.concatenate([np.ones((ell - 1) * N), mu ** ell / (mu ** ell - alpha)])
                             .astype(complex))
    assert np.abs(ev - expect).max() < 1e-8
    assert ev.real.max() == pytest.approx(1.0 / (1.0 - alpha), rel=1e-9)
    assert ev.real.min() == pytest.approx(1.0, abs=1e-9)
    # Remark after Thm thm:evals: max |lam - 1| <= alpha/(1 - eta) for alpha <= eta < 1
    eta = max(alpha, 0.95)
    assert np.abs(ev - 1).max() <= alpha / (1 - eta) + 1e-9


def test_gamma_condition():
    g = GOLD["fig2_kappa"]
    assert math.log10(circ.gamma_condition(g["ell"], g["alpha"])) == pytest.approx(g["log10"], abs=1e-12)
    for ell, alpha in [(4, 0.1), (10, 1e-4)]:
        s = np.linalg.svd(_F(ell) @ np.diag(circ.gammas(ell, alpha)), compute_uv=False)
        assert s.max() / s.min() == pytest.approx(alpha ** (-(ell - 1) / ell), rel=1e-10)
        assert circ.gamma_condition(ell, alpha) == pytest.approx(s.max() / s.min(), rel=1e-10)
