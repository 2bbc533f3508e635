"""Saddle-point inner solver P_SP (oracle; test infrastructure only).

PAPER.md §4 (lines 556-618) and §5.1 (lines 694-697):
  * complex block problems (A - lam I) x = b are rewritten as the real system
    Eq. (eq:saddlesystem)  [[Im lam I, A - Re lam I], [A - Re lam I, -Im lam I]]
    [Re x; -Im x] = [-Im b; Re b], solved by MINRES preconditioned with
    P_D = diag(Phi + Psi, Phi + Psi) (Eq. eq:minresprecond), Phi = Im lam I,
    Psi = A - Re lam I; Phi SPD needs Im lam > 0, so blocks with Im Lambda_k < 0
    are conjugated first (reading R16);
  * the two real shifts are solved by PCG;
  * (Phi + Psi)^{-1} and (A - Lambda I)^{-1} are approximated by ONE multigrid
    V-cycle each. The paper uses HSL_MI20 AMG (out of scope, not in the
    container); reading R16 replaces it by a geometric V(1,1) cycle: damped
    Jacobi (omega = 0.8), cell aggregation of 2 per axis with piecewise-constant
    P and Galerkin coarse operators P^T A P, dense solve once every axis <= 8;
  * fixed k_in iterations, no inner tolerance (BASELINE.json configs[3]).
Matvec accounting (Table 1): 2 per MINRES iteration, 1 per PCG iteration.
"""
from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp

from . import circulant as circ
from . import operator as op

OMEGA = 0.8
COARSEST_MAX_AXIS = 8


def saddle_dense(A: np.ndarray, lam: complex) -> np.ndarray:
    """Dense 2N x 2N assembly of Eq. (eq:saddlesystem)."""
    N = A.shape[0]
    I = np.eye(N)
    Psi = A - lam.real * I
    return np.block([[lam.imag * I, Psi], [Psi, -lam.imag * I]])


def saddle_apply(w: op.Weights, lam: complex, uv):
    """S [u; v] = [Im lam u + Psi v; Psi u - Im lam v] (two A applications)."""
    N = w.N
    u = uv[:N].reshape(w.shape)
    v = uv[N:].reshape(w.shape)
    Av = op.apply_A(w, v) - lam.real * v
    Au = op.apply_A(w, u) - lam.real * u
    return np.concatenate([(lam.imag * u + Av).ravel(), (Au - lam.imag * v).ravel()])


# ----------------------------------------------------------------------------- multigrid
class Level:
    def __init__(self, shape, A0: sp.csr_matrix, cnt: np.ndarray):
        self.shape = shape           # (nz, ny, nx)
        self.A0 = A0                 # Galerkin image of A (shift 0)
        self.cnt = cnt               # Galerkin image of I (diagonal: fine cells per aggregate)
        self.P = None                # prolongation to this level from the next coarser

    def A(self, s: float) -> sp.csr_matrix:
        return (self.A0 + sp.diags(s * self.cnt)).tocsr()


def _coarse_shape(shape):
    return tuple(1 if n == 1 else (n + 1) // 2 for n in shape)


def _aggregation(shape):
    nz, ny, nx = shape
    cz, cy, cx = _coarse_shape(shape)
    k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    agg = ((k // 2 if nz > 1 else k) * cy + (j // 2 if ny > 1 else j)) * cx + \
        (i // 2 if nx > 1 else i)
    Nf = nz * ny * nx
    return sp.csr_matrix((np.ones(Nf), (np.arange(Nf), agg.ravel())), shape=(Nf, cz * cy * cx))


def hierarchy(w: op.Weights):
    """Levels 0..L: A_{l+1} = P_l^T A_l P_l (Galerkin), stop when every axis <= 8."""
    levels = [Level(w.shape, op.sparse_A(w), np.ones(w.N))]
    while max(levels[-1].shape) > COARSEST_MAX_AXIS:
        f = levels[-1]
        P = _aggregation(f.shape)
        f.P = P
        A0 = (P.T @ f.A0 @ P).tocsr()
        cnt = P.T @ f.cnt
        levels.append(Level(_coarse_shape(f.shape), A0, np.asarray(cnt).ravel()))
    return levels


def vcycle(levels, s: float, b, l: int = 0):
    """One V(1,1) cycle for (A + s I) x = b from x = 0 (symmetric, SPD for omega < 1)."""
    lev = levels[l]
    A = lev.A(s)
    if l == len(levels) - 1:
        return np.linalg.solve(A.toarray(), b)
    D = A.diagonal()
    x = OMEGA * b / D                       # pre-smoothing from zero
    r = b - A @ x
    xc = vcycle(levels, s, lev.P.T @ r, l + 1)
    x = x + lev.P @ xc
    x = x + OMEGA * (b - A @ x) / D         # post-smoothing
    return x


# ----------------------------------------------------------------------------- Krylov
def minres(apply_S, apply_M, b, k: int):
    """Preconditioned MINRES, k iterations from x_0 = 0 (Elman-Silvester-Wathen,
    Alg. 2.4 form; M symmetric positive definite)."""
    x = np.zeros_like(b)
    v_prev = np.zeros_like(b)
    v = b.copy()
    z = apply_M(v)
    gamma = math.sqrt(max(float(np.dot(z, v)), 0.0))
    if gamma == 0.0:
        return x
    gamma_prev = 1.0
    eta = gamma
    s_prev, s_cur = 0.0, 0.0
    c_prev, c_cur = 1.0, 1.0
    w_prev = np.zeros_like(b)
    w_cur = np.zeros_like(b)
    for _j in range(k):
        z = z / gamma
        Sz = apply_S(z)
        delta = float(np.dot(Sz, z))
        v_next = Sz - (delta / gamma) * v - (gamma / gamma_prev) * v_prev
        z_next = apply_M(v_next)
        gamma_next = math.sqrt(max(float(np.dot(z_next, v_next)), 0.0))
        a0 = c_cur * delta - c_prev * s_cur * gamma
        a1 = math.sqrt(a0 * a0 + gamma_next * gamma_next)
        a2 = s_cur * delta + c_prev * c_cur * gamma
        a3 = s_prev * gamma
        c_next = a0 / a1
        s_next = gamma_next / a1
        w_next = (z - a3 * w_prev - a2 * w_cur) / a1
        x = x + c_next * eta * w_next
        eta = -s_next * eta
        if gamma_next == 0.0:
            break
        v_prev, v = v, v_next
        z = z_next
        gamma_prev, gamma = gamma, gamma_next
        w_prev, w_cur = w_cur, w_next
        s_prev, s_cur = s_cur, s_next
        c_prev, c_cur = c_cur, c_next
    return x


def pcg(apply_A, apply_M, b, k: int):
    """Preconditioned CG (Hestenes-Stiefel), k iterations from x_0 = 0."""
    x = np.zeros_like(b)
    r = b.copy()
    z = apply_M(r)
    p = z.copy()
    rho = float(np.dot(r, z))
    for i in range(k):
        if rho == 0.0:
            break
        q = apply_A(p)
        a = rho / float(np.dot(p, q))
        x = x + a * p
        r = r - a * q
        if i == k - 1:
            break
        z = apply_M(r)
        rho_new = float(np.dot(r, z))
        p = z + (rho_new / rho) * p
        rho = rho_new
    return x


def sp_apply(w: op.Weights, r, ell: int, alpha: float, k: int, levels=None):
    """P_SP^{-1} r: Eq. (eq:Paform) with every block problem solved by k iterations of
    MINRES on the saddle system (complex Lambda_k) or PCG (real Lambda_k)."""
    if levels is None:
        levels = hierarchy(w)
    N = w.N
    r = np.asarray(r).reshape((ell,) + w.shape)
    what = circ.forward(r, ell, alpha)
    lam = circ.shifts(ell, alpha)
    yhat = np.empty_like(what)
    for kk in range(ell):
        bk = what[kk].reshape(-1)
        if kk == 0 or 2 * kk == ell:        # real shift: PCG on A - Lambda I
            s = -lam[kk].real
            x = pcg(lambda v, s=s: op.apply_A(w, v).reshape(-1) + s * v,
                    lambda v, s=s: vcycle(levels, s, v), bk.real.copy(), k)
            yhat[kk] = x.reshape(w.shape)
            continue
        flip = lam[kk].imag < 0
        lk = np.conj(lam[kk]) if flip else lam[kk]
        bb = np.conj(bk) if flip else bk
        s = lk.imag - lk.real                # Phi + Psi = A + (Im lam - Re lam) I
        rhs = np.concatenate([-bb.imag, bb.real])

        def M(uv, s=s):
            return np.concatenate([vcycle(levels, s, uv[:N]), vcycle(levels, s, uv[N:])])

        uv = minres(lambda t, lk=lk: saddle_apply(w, lk, t), M, rhs, k)
        x = uv[:N] - 1j * uv[N:]
        yhat[kk] = (np.conj(x) if flip else x).reshape(w.shape)
    return circ.inverse(yhat, ell, alpha)
