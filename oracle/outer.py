"""The paper's outer solver: Chebyshev semi-iteration on the left-preconditioned all-at-once
system (oracle; test infrastructure only).

PAPER.md:102-107 Eq. (eq:precondsystem): CI applied to P^{-1} calA x = P^{-1} b, foci from
Cor. cor:extremeevals: lambda in [1, mu_N^ell / (mu_N^ell - alpha)], mu_N
the smallest eigenvalue of A, NOT adjusted for the approximate preconditioners.
Unpreconditioned (P = I): foci = the extreme eigenvalues of A, which are those of calA (block
lower triangular with A on the diagonal).
PAPER.md:647: initial guess chi_0 = 0, stop when r_p = ||b - calA chi_p||_2 / ||b||_2 < 1e-6;
the reported count is p (= the number of P^{-1} applications). SPEC.md:375-383 solve_outer.
The recurrence is the same three-term Chebyshev acceleration as the inner solves (reading R8),
driven by the preconditioned residual z_p = P^{-1}(b - calA chi_p):
    chi_1 = chi_0 + z_0/theta, rho_0 = delta/theta,
    rho_p = 1/(2 theta/delta - rho_{p-1}),
    chi_{p+1} = chi_p + rho_p rho_{p-1} (chi_p - chi_{p-1}) + (2 rho_p/delta) z_p,
    theta = (l_max + l_min)/2, delta = (l_max - l_min)/2.
"""
from __future__ import annotations

import dataclasses

import numpy as np


@dataclasses.dataclass
class CiResult:
    x: np.ndarray
    iters: int
    converged: bool
    history: list             # r_p for p = 0..iters


def extreme_eigs(mu_min: float, ell: int, alpha: float):
    """Cor. cor:extremeevals: (1, mu_min^ell / (mu_min^ell - alpha)) for 0 < alpha < mu_min^ell."""
    m = mu_min ** ell
    return 1.0, m / (m - alpha)


def ci_outer(apply_op, apply_prec, b, l_min: float, l_max: float, tol: float = 1e-6,
             maxit: int = 5000) -> CiResult:
    b = np.asarray(b, dtype=np.float64)
    shape = b.shape
    bv = b.reshape(-1)
    nb = np.linalg.norm(bv)
    x_prev = np.zeros_like(bv)
    x = np.zeros_like(bv)
    r = bv.copy()
    hist = [1.0]
    if nb == 0.0:
        return CiResult(x.reshape(shape), 0, True, hist)
    theta = 0.5 * (l_max + l_min)
    delta = 0.5 * (l_max - l_min)
    rho = None
    for p in range(maxit):
        if np.linalg.norm(r) < tol * nb:
            return CiResult(x.reshape(shape), p, True, hist)
        z = r if apply_prec is None else np.asarray(apply_prec(r.reshape(shape))).reshape(-1)
        if p == 0:
            x_new = x + z / theta
            rho = delta / theta
        else:
            rho_new = 1.0 / (2.0 * theta / delta - rho)
            x_new = x + rho_new * rho * (x - x_prev) + (2.0 * rho_new / delta) * z
            rho = rho_new
        x_prev, x = x, x_new
        r = bv - np.asarray(apply_op(x.reshape(shape))).reshape(-1)
        hist.append(np.linalg.norm(r) / nb)
    return CiResult(x.reshape(shape), maxit, False, hist)
