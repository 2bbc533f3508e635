"""Flexible GMRES with CGS2 orthogonalisation (oracle; test infrastructure only).

Not in the paper: BASELINE.json:north_star mandates right-preconditioned GMRES at
rtol 1e-10 instead of the paper's outer CI. Reading R1/R14/R15
(DESIGN.md): FGMRES, x_0 = 0, unrestarted, CGS2 (two classical Gram-Schmidt
passes), Givens r = hypot(h_jj, h_{j+1,j}), c = h_jj/r, s = h_{j+1,j}/r, stop when
|g_{j+1}| <= rtol * ||b|| after every Arnoldi step; happy breakdown stops too.
Iteration count = number of preconditioner applications.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np


@dataclasses.dataclass
class GmresResult:
    x: np.ndarray
    iters: int
    converged: bool
    relres_est: float
    history: list


def fgmres(apply_op, apply_prec, b, rtol: float = 1e-10, maxit: int = 200) -> GmresResult:
    b = np.asarray(b, dtype=np.float64)
    shape = b.shape
    bv = b.reshape(-1)
    beta = float(np.sqrt(np.dot(bv, bv)))
    if beta == 0.0:
        return GmresResult(np.zeros_like(b), 0, True, 0.0, [])
    V = [bv / beta]
    Z = []
    H = np.zeros((maxit + 1, maxit))
    cs = np.zeros(maxit)
    sn = np.zeros(maxit)
    g = np.zeros(maxit + 1)
    g[0] = beta
    hist = []
    converged = False
    m = 0
    for j in range(maxit):
        z = np.asarray(apply_prec(V[j].reshape(shape))).reshape(-1)
        Z.append(z)
        w = np.asarray(apply_op(z.reshape(shape))).reshape(-1).copy()
        h1 = np.array([np.dot(V[i], w) for i in range(j + 1)])      # CGS pass 1
        for i in range(j + 1):
            w -= h1[i] * V[i]
        h2 = np.array([np.dot(V[i], w) for i in range(j + 1)])      # CGS pass 2
        for i in range(j + 1):
            w -= h2[i] * V[i]
        H[:j + 1, j] = h1 + h2
        hn = float(np.sqrt(np.dot(w, w)))
        H[j + 1, j] = hn
        for i in range(j):                                          # old rotations
            t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
            H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
            H[i, j] = t
        r = math.hypot(H[j, j], H[j + 1, j])
        cs[j] = H[j, j] / r
        sn[j] = H[j + 1, j] / r
        H[j, j] = r
        H[j + 1, j] = 0.0
        g[j + 1] = -sn[j] * g[j]
        g[j] = cs[j] * g[j]
        m = j + 1
        rel = abs(g[j + 1]) / beta
        hist.append(rel)
        if hn == 0.0 or rel <= rtol:
            converged = True
            break
        V.append(w / hn)
    y = np.zeros(m)
    for i in range(m - 1, -1, -1):                                  # back substitution
        y[i] = (g[i] - np.dot(H[i, i + 1:m], y[i + 1:m])) / H[i, i]
    x = np.zeros_like(bv)
    for i in range(m):
        x += y[i] * Z[i]
    return GmresResult(x.reshape(shape), m, converged, hist[-1] if hist else 0.0, hist)
