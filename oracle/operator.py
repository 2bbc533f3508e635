"""Spatial operator A and the all-at-once operator  (oracle; test infrastructure only).

A = I + c * (-div kappa grad)_h on a cell-centred grid with zero-flux (Neumann)
boundaries, the BASELINE.json operator (reading R2/R3):

    (A u)_P = u_P + sum_{interior faces f of P} w_f (u_P - u_nb(f)),
    w_f = c * kappa_f / h_a^2  (h_a = 1/n_a for the face's axis a).

The all-at-once operator is PAPER.md:35-46 Eq. (eq:A):
    calA = I_ell (x) A - Sigma (x) I_N,   Sigma = lower block shift,
i.e. y_1 = A x_1, y_j = A x_j - x_{j-1}.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla


class Weights:
    """Face weights w_f = c*kappa_f*n_a^2 in natural interior layout.

    bd = (bx, by, bz): Dirichlet boundary-face weights per axis (the paper's own operator,
    PAPER.md:630-637 Eq. IminusLap: a boundary face to a zero ghost value adds bd_a * u_P to
    (A u)_P); (0, 0, 0) -- the default -- is the BASELINE zero-flux Neumann operator."""

    def __init__(self, shape, c, kx, ky, kz, bd=(0.0, 0.0, 0.0)):
        nz, ny, nx = shape
        self.shape = (nz, ny, nx)
        self.wx = c * float(nx) ** 2 * np.asarray(kx, dtype=np.float64).reshape(nz, ny, nx - 1)
        self.wy = c * float(ny) ** 2 * np.asarray(ky, dtype=np.float64).reshape(nz, ny - 1, nx)
        self.wz = c * float(nz) ** 2 * np.asarray(kz, dtype=np.float64).reshape(nz - 1, ny, nx)
        self.bd = tuple(float(v) for v in bd)

    @property
    def N(self):
        nz, ny, nx = self.shape
        return nz * ny * nx


def weights(prob) -> Weights:
    return Weights(prob.shape, prob.c, prob.kx, prob.ky, prob.kz, getattr(prob, "bd", (0.0, 0.0, 0.0)))


def boundary_diag(w: Weights) -> np.ndarray:
    """Per-cell Dirichlet term: sum of bd_a over the cell's faces on the domain boundary
    (zero for the Neumann operator)."""
    d = np.zeros(w.shape)
    bx, by, bz = getattr(w, "bd", (0.0, 0.0, 0.0))
    nz, ny, nx = w.shape
    for axis, b, n in ((2, bx, nx), (1, by, ny), (0, bz, nz)):
        if b == 0.0 or n == 1:
            continue
        lo = [slice(None)] * 3
        hi = [slice(None)] * 3
        lo[axis] = 0
        hi[axis] = n - 1
        d[tuple(lo)] += b
        d[tuple(hi)] += b
    return d


def apply_A(w: Weights, u):
    """(A u)_P = u_P + sum_f w_f (u_P - u_nb); u shaped (nz, ny, nx), real or complex."""
    u = np.asarray(u).reshape(w.shape)
    out = u.copy()
    d = u[:, :, 1:] - u[:, :, :-1]            # across x-faces
    out[:, :, :-1] -= w.wx * d
    out[:, :, 1:] += w.wx * d
    d = u[:, 1:, :] - u[:, :-1, :]            # across y-faces
    out[:, :-1, :] -= w.wy * d
    out[:, 1:, :] += w.wy * d
    d = u[1:, :, :] - u[:-1, :, :]            # across z-faces
    out[:-1, :, :] -= w.wz * d
    out[1:, :, :] += w.wz * d
    if any(getattr(w, "bd", (0.0, 0.0, 0.0))):  # Dirichlet faces: zero ghost values
        out = out + boundary_diag(w) * u
    return out


def gershgorin_max(w: Weights) -> float:
    """mu_max bound = max_P (1 + 2 sum_{f in P} w_f)  (reading R5)."""
    s = np.zeros(w.shape)
    s[:, :, :-1] += w.wx
    s[:, :, 1:] += w.wx
    s[:, :-1, :] += w.wy
    s[:, 1:, :] += w.wy
    s[:-1, :, :] += w.wz
    s[1:, :, :] += w.wz
    return float(np.max(1.0 + 2.0 * s + boundary_diag(w)))


def incidence(shape):
    """Face-difference matrix G (one row per interior face, +1 at the upper cell,
    -1 at the lower cell) and the list of face axes, in x, y, z face order."""
    nz, ny, nx = shape
    idx = np.arange(nz * ny * nx).reshape(shape)
    rows, cols, vals = [], [], []
    nf = 0
    for lo, hi in ((idx[:, :, :-1], idx[:, :, 1:]), (idx[:, :-1, :], idx[:, 1:, :]),
                   (idx[:-1, :, :], idx[1:, :, :])):
        m = lo.size
        f = np.arange(nf, nf + m)
        rows += [f, f]
        cols += [hi.ravel(), lo.ravel()]
        vals += [np.ones(m), -np.ones(m)]
        nf += m
    G = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(nf, nz * ny * nx))
    return G


def sparse_A(w: Weights) -> sp.csr_matrix:
    """Independent assembly A = I + G^T diag(w) G (graph Laplacian form)."""
    G = incidence(w.shape)
    wf = np.concatenate([w.wx.ravel(), w.wy.ravel(), w.wz.ravel()])
    return (sp.identity(w.N, format="csr") + G.T @ sp.diags(wf) @ G
            + sp.diags(boundary_diag(w).ravel())).tocsr()


def dense_A(w: Weights) -> np.ndarray:
    return sparse_A(w).toarray()


def apply_allatonce(w: Weights, x):
    """PAPER.md:35-46 Eq. (eq:A): y_1 = A x_1, y_j = A x_j - x_{j-1}."""
    x = np.asarray(x)
    ell = x.shape[0]
    x = x.reshape((ell,) + w.shape)
    y = np.empty_like(x)
    for j in range(ell):
        y[j] = apply_A(w, x[j])
        if j > 0:
            y[j] -= x[j - 1]
    return y


def dense_allatonce(A: np.ndarray, ell: int) -> np.ndarray:
    """calA = I_ell (x) A + Sigma (x) (-I_N) built with Kronecker products."""
    N = A.shape[0]
    Sigma = np.eye(ell, k=-1)
    return np.kron(np.eye(ell), A) - np.kron(Sigma, np.eye(N))


def solve_recurrence(w: Weights, b):
    """x* = calA^{-1} b by the sequential recurrence x_1 = A^{-1} b_1,
    x_j = A^{-1}(b_j + x_{j-1}) (the ell-step form)."""
    b = np.asarray(b)
    ell = b.shape[0]
    lu = spla.splu(sparse_A(w).tocsc())
    x = np.empty((ell,) + w.shape, dtype=np.result_type(b.dtype, np.float64))
    prev = np.zeros(w.N)
    for j in range(ell):
        prev = lu.solve(b[j].reshape(-1) + prev)
        x[j] = prev.reshape(w.shape)
    return x
