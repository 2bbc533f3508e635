"""Varying diagonal blocks A_1..A_ell (oracle, test infrastructure only).

PAPER.md:991 (Conclusions): "the block alpha-circulant preconditioner can be extended to a
problem with similar block structure, with varying diagonal blocks A_1, A_2, ..., A_ell using
some 'representative' or average choice A_hat ... The methods and theory of Sections 3 and 4
apply directly in this setting. However, the eigenvalue bounds on the preconditioned system
... no longer hold, making the use of this preconditioner within Chebyshev semi-iteration
challenging or impossible."

So (reading R26):
    calA_var = blockdiag(A_1, ..., A_ell) - Sigma (x) I_N        (y_j = A_j x_j - x_{j-1}),
    A_hat    = (1/ell) sum_j A_j = I + c(-div kappa_hat grad)_h with kappa_hat = mean_j kappa_j
               (A is affine in the face weights, so the average operator is the operator of the
               averaged weights),
    P_alpha(A_hat) applied exactly as before (nested Chebyshev / saddle point), GMRES outside
    (CI needs the eigenvalue bounds that no longer hold). Parity unpinned by the paper: it
    prints no numbers for this setting; the pins below are definitions and identities.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse.linalg as spla

from . import operator as op


def block_weights(prob_blocks) -> list:
    """Face weights of every block: prob_blocks.kx_blocks[j] etc. (synth.make_varying_problem)."""
    p = prob_blocks
    return [op.Weights(p.shape, p.c, p.kx_blocks[j], p.ky_blocks[j], p.kz_blocks[j]) for j in range(p.ell)]


def mean_weights(ws) -> op.Weights:
    """Face weights of A_hat = mean_j A_j (the mean of the face weights)."""
    w = op.Weights.__new__(op.Weights)
    w.shape = ws[0].shape
    w.wx = np.mean([v.wx for v in ws], axis=0)
    w.wy = np.mean([v.wy for v in ws], axis=0)
    w.wz = np.mean([v.wz for v in ws], axis=0)
    w.bd = ws[0].bd
    return w


def apply_allatonce_var(ws, x):
    """y_1 = A_1 x_1, y_j = A_j x_j - x_{j-1} (PAPER.md:35-46 with varying diagonal blocks)."""
    x = np.asarray(x)
    ell = len(ws)
    x = x.reshape((ell,) + ws[0].shape)
    y = np.empty_like(x)
    for j in range(ell):
        y[j] = op.apply_A(ws[j], x[j])
        if j > 0:
            y[j] -= x[j - 1]
    return y


def solve_recurrence_var(ws, b):
    """x* by the sequential recurrence x_1 = A_1^{-1} b_1, x_j = A_j^{-1}(b_j + x_{j-1})."""
    b = np.asarray(b)
    ell = len(ws)
    x = np.empty((ell,) + ws[0].shape)
    prev = np.zeros(ws[0].N)
    for j in range(ell):
        prev = spla.spsolve(op.sparse_A(ws[j]).tocsc(), b[j].reshape(-1) + prev)
        x[j] = prev.reshape(ws[0].shape)
    return x
