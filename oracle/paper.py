"""The paper's own test operator (oracle; test infrastructure only).

PAPER.md:630-637 §5 Eq. (IminusLap): A = I_N - (nu/h^2) L, 2D Dirichlet 5-point
Laplacian on the n_x x n_x interior vertices of the unit square, h = 1/(n_x+1),
nu = D^2/(2 ell - 4), D = 0.2.
PAPER.md:998-1020 Appendix A: mu_{i,j} = 1 + (4 nu/h^2)(sin^2(i pi/(2(n_x+1))) +
sin^2(j pi/(2(n_x+1)))); mu_min = mu_{1,1}, mu_max = mu_{n_x,n_x}.
Used by the Algorithm 1 pins against Tables 3, 4 and 8 (paper-operator mode,
SURVEY.md §8(f) N1).
"""
from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp

from . import operator as op


def nu(ell: int, D: float = 0.2) -> float:
    return D * D / (2.0 * ell - 4.0)


def bounds(nx: int, ell: int, D: float = 0.2):
    """(mu_min, mu_max) of Appendix A."""
    h = 1.0 / (nx + 1)
    a = 8.0 * nu(ell, D) / (h * h)
    lo = 1.0 + a * math.sin(math.pi / (2 * (nx + 1))) ** 2
    hi = 1.0 + a * math.sin(nx * math.pi / (2 * (nx + 1))) ** 2
    return lo, hi


def eigenvalues(nx: int, ell: int, D: float = 0.2) -> np.ndarray:
    h = 1.0 / (nx + 1)
    i = np.arange(1, nx + 1)
    s = np.sin(i * math.pi / (2 * (nx + 1))) ** 2
    return (1.0 + 4.0 * nu(ell, D) / (h * h) * (s[:, None] + s[None, :])).ravel()


def sparse_A(nx: int, ell: int, D: float = 0.2) -> sp.csr_matrix:
    """Eq. (IminusLap) assembled with the standard 5-point Dirichlet Laplacian."""
    h = 1.0 / (nx + 1)
    T = sp.diags([np.ones(nx - 1), -2.0 * np.ones(nx), np.ones(nx - 1)], [-1, 0, 1])
    L = sp.kron(sp.identity(nx), T) + sp.kron(T, sp.identity(nx))
    return (sp.identity(nx * nx) - (nu(ell, D) / (h * h)) * L).tocsr()


def weights(nx: int, ell: int, D: float = 0.2) -> op.Weights:
    """Eq. (IminusLap) in face-weight form: every interior face and every boundary face
    (to a zero Dirichlet ghost) of the n_x x n_x vertex grid carries nu/h^2, h = 1/(n_x+1)."""
    w = op.Weights.__new__(op.Weights)
    w.shape = (1, nx, nx)
    f = nu(ell, D) * (nx + 1) ** 2
    w.wx = np.full((1, nx, nx - 1), f)
    w.wy = np.full((1, nx - 1, nx), f)
    w.wz = np.zeros((0, nx, nx))
    w.bd = (f, f, 0.0)
    return w
