"""Nested Chebyshev semi-iteration preconditioners P_NC1 / P_NC2 (oracle; test infrastructure only).

PAPER.md §3 (lines 286-446): CI applied to B_k = A - Lambda_k I whose spectrum lies
on the segment S_k = [mu_min - Lambda_k, mu_max - Lambda_k] parallel to the real
axis (Lemma lem:evals). CI takes the shifted-and-scaled Chebyshev polynomial
(Prop. prop:errorbound):
    e_p = T_p((theta - B)/delta) / T_p(theta/delta) e_0,
    theta = (mu_max + mu_min)/2 - Lambda_k (complex),  delta = (mu_max - mu_min)/2.
The paper never writes the recurrence (reading R8); we use the standard
three-term Chebyshev-acceleration recurrence, whose iterates satisfy exactly
the polynomial contract above (pinned in tests/test_oracle_chebyshev.py):
    x_0 = 0, x_1 = b/theta, rho_0 = delta/theta,
    rho_s = 1/(2 theta/delta - rho_{s-1}),
    x_{s+1} = x_s + rho_s rho_{s-1} (x_s - x_{s-1}) + (2 rho_s/delta)(b - B x_s).
"k iterations" = the iterate x_k (reading R9): k-1 applications of B.
"""
from __future__ import annotations

import math

import numpy as np

from . import circulant as circ
from . import operator as op


def ci_solve(apply_B, b, theta: complex, delta: float, p: int):
    """Return x_p, the p-th Chebyshev iterate for B x = b from x_0 = 0."""
    if p < 1:
        raise ValueError("p >= 1")
    x_prev = np.zeros_like(b)
    x = b / theta
    if delta == 0.0:            # single-point spectrum: B = theta I, x_1 is exact (R10)
        return x
    rho_prev = delta / theta
    for _s in range(1, p):
        rho = 1.0 / (2.0 * theta / delta - rho_prev)
        x_next = x + rho * rho_prev * (x - x_prev) + (2.0 * rho / delta) * (b - apply_B(x))
        x_prev, x, rho_prev = x, x_next, rho
    return x


def ci_iterations_to_tol(apply_B, b, theta: complex, delta: float, tol: float, pmax: int):
    """Smallest p with ||b - B x_p|| / ||b|| < tol (relative residual, PAPER.md:647 stopping
    rule applied to one block problem, as in Table 2 tab:Cheb conv tol)."""
    nb = np.linalg.norm(b)
    x_prev = np.zeros_like(b)
    x = b / theta
    rho_prev = delta / theta
    for p in range(1, pmax + 1):
        res = b - apply_B(x)
        if np.linalg.norm(res) < tol * nb:
            return p
        rho = 1.0 / (2.0 * theta / delta - rho_prev)
        x_next = x + rho * rho_prev * (x - x_prev) + (2.0 * rho / delta) * res
        x_prev, x, rho_prev = x, x_next, rho
    return None


def ci_coefficients(theta: complex, delta: float, p: int):
    """(a_s, b_s) = (rho_s rho_{s-1}, 2 rho_s/delta) for s = 1..p-1 (host tables)."""
    out = []
    rho_prev = delta / theta
    for _s in range(1, p):
        rho = 1.0 / (2.0 * theta / delta - rho_prev)
        out.append((rho * rho_prev, 2.0 * rho / delta))
        rho_prev = rho
    return out


def sigma_bound(mu_min: float, mu_max: float, re_lam: float) -> float:
    """Thm thm:convergence: rho(lambda) < sigma =
    (sqrt(kappa)-1)/(sqrt(kappa)+1), kappa = kappa(Re B) = (mu_max - Re lam)/(mu_min - Re lam)."""
    kap = (mu_max - re_lam) / (mu_min - re_lam)
    s = math.sqrt(kap)
    return (s - 1.0) / (s + 1.0)


def p_star(vmin: float, vmax: float, eps: float) -> float:
    """Thm thm:AxelssonIteration: a-priori CI iteration count."""
    r = math.sqrt(vmin / vmax)
    num = math.log(1.0 / eps + math.sqrt(1.0 / eps ** 2 - 1.0))
    return num / math.log((1.0 + r) / (1.0 - r))


def re_shift(ell: int, alpha: float, k: int) -> float:
    """Re Lambda_k evaluated from the reduced angle min(k, ell-k) so that conjugate
    pairs get bit-identical values (reading R11)."""
    kk = min(k, ell - k)
    return alpha ** (1.0 / ell) * math.cos(2.0 * math.pi * kk / ell)


def allocate(ell: int, mu_min: float, mu_max: float, alpha: float, budget, method: str,
             k_uniform=None):
    """Inner iteration counts per block k = 0..ell-1.

    NC1: every block gets the same count (k_uniform).
    NC2 = Algorithm 1: sigma_j from Thm 3.6, r(j) = ln sigma_1 /
    ln sigma_j, normalise, all = floor(r * budget) entrywise; then clamp >= 1 (R11).
    `budget` is the paper's ell*n_x*eta or, for BASELINE's fixed k, ell*k.
    """
    if method == "nc1":
        return [int(k_uniform)] * ell
    if method != "nc2":
        raise ValueError(method)
    if mu_max == mu_min:                       # delta = 0: every block is exact at p=1
        return [max(1, int(math.floor(budget / ell)))] * ell
    sig = [sigma_bound(mu_min, mu_max, re_shift(ell, alpha, k)) for k in range(ell)]
    r = [math.log(sig[0]) / math.log(s) for s in sig]
    tot = sum(r)
    r = [x / tot for x in r]
    return [max(1, int(math.floor(x * budget))) for x in r]


def nc_apply(w: op.Weights, r, ell: int, alpha: float, mu_min: float, mu_max: float,
             alloc):
    """P_NC^{-1} r: Eq. (eq:Paform) with every block problem (A - Lambda_k) y_k = hat w_k
    (Eq. eq:blockproblem) solved approximately by alloc[k] CI iterations."""
    r = np.asarray(r).reshape((ell,) + w.shape)
    what = circ.forward(r, ell, alpha)
    lam = circ.shifts(ell, alpha)
    delta = 0.5 * (mu_max - mu_min)
    yhat = np.empty_like(what)
    for k in range(ell):
        theta = 0.5 * (mu_max + mu_min) - lam[k]
        lk = lam[k]
        yhat[k] = ci_solve(lambda v, lk=lk: op.apply_A(w, v) - lk * v, what[k],
                           theta, delta, int(alloc[k]))
    return circ.inverse(yhat, ell, alpha)


def nc_apply_f32(w: op.Weights, r, ell: int, alpha: float, mu_min: float, mu_max: float, alloc):
    """Mixed-precision P_NC^{-1} r (fp32 inner sweeps, fp64 outer): nc_apply with
    every block's CI recurrence evaluated in single precision -- the transformed right-hand side,
    the face weights and the iterates in complex64 / float32, the scalars theta, delta, rho_s
    computed in fp64 and rounded to fp32 -- and the transforms in fp64. Parity unpinned by the
    paper (it names the setting only); pinned against nc_apply to fp32 accuracy."""
    r = np.asarray(r).reshape((ell,) + w.shape)
    what = circ.forward(r, ell, alpha)
    lam = circ.shifts(ell, alpha)
    delta = 0.5 * (mu_max - mu_min)
    w32 = op.Weights.__new__(op.Weights)
    w32.shape = w.shape
    w32.wx, w32.wy, w32.wz = (np.asarray(a, dtype=np.float32) for a in (w.wx, w.wy, w.wz))
    w32.bd = tuple(np.float32(v) for v in getattr(w, "bd", (0.0, 0.0, 0.0)))
    yhat = np.empty_like(what)
    for k in range(ell):
        theta = 0.5 * (mu_max + mu_min) - lam[k]
        lk = np.complex64(lam[k])
        b = what[k].astype(np.complex64)
        p = int(alloc[k])
        x_prev = np.zeros_like(b)
        x = (b * np.complex64(1.0 / theta)).astype(np.complex64)
        if delta > 0.0:
            rho_prev = delta / theta
            for _s in range(1, p):
                rho = 1.0 / (2.0 * theta / delta - rho_prev)
                a_s, b_s = np.complex64(rho * rho_prev), np.complex64(2.0 * rho / delta)
                res = b - (op.apply_A(w32, x).astype(np.complex64) - lk * x)
                x_next = x + a_s * (x - x_prev) + b_s * res
                x_prev, x, rho_prev = x, x_next.astype(np.complex64), rho
        yhat[k] = x.astype(np.complex128)
    return circ.inverse(yhat, ell, alpha)
