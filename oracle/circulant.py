"""Block alpha-circulant preconditioner in Kronecker/DFT form (oracle; test infrastructure only).

PAPER.md:59-76 Eq. (eq:exactPBE):  P_alpha = I_ell (x) A + C_alpha (x) (-I_N),
C_alpha = lower shift with alpha in the top-right corner.
PAPER.md:229-254 Eqs. (eq:palpha), (eq:Paform):
    P_alpha^{-1} = (Gamma^{-1} U (x) I)(I (x) A - Lambda (x) I)^{-1}(U^* Gamma (x) I),
    Gamma_alpha = diag(1, alpha^{1/ell}, ..., alpha^{(ell-1)/ell}).

Reading R6: the printed pairing of U's columns with
lambda_j = alpha^{1/ell} e^{+2 pi i (j-1)/ell} does not reproduce C_alpha
(pinned by tests/test_oracle_circulant.py::test_printed_pairing_fails).  The
consistent pairing, used here, is forward transform U^* = F with
F_{kj} = ell^{-1/2} e^{-2 pi i j k/ell}, shift Lambda_k = alpha^{1/ell} e^{-2 pi i k/ell}
(= conj of the paper's lambda_{k+1}; same multiset), inverse U = F^*.
Indices are 0-based: block j = 0..ell-1, frequency k = 0..ell-1.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from . import operator as op


def gammas(ell: int, alpha: float) -> np.ndarray:
    """gamma_j = alpha^{j/ell}, j = 0..ell-1 (reading R7)."""
    return np.array([alpha ** (j / ell) for j in range(ell)])


def shifts(ell: int, alpha: float) -> np.ndarray:
    """Lambda_k = alpha^{1/ell} exp(-2 pi i k / ell) (PAPER.md:242 with reading R6)."""
    k = np.arange(ell)
    return alpha ** (1.0 / ell) * np.exp(-2j * np.pi * k / ell)


def paper_roots(ell: int, alpha: float) -> np.ndarray:
    """The paper's labelling lambda_j = alpha^{1/ell} e^{2 pi i (j-1)/ell}, j=1..ell
    (Fig. 1 anticlockwise from lambda_1 = alpha^{1/ell})."""
    j = np.arange(1, ell + 1)
    return alpha ** (1.0 / ell) * np.exp(2j * np.pi * (j - 1) / ell)


def C_alpha(ell: int, alpha: float) -> np.ndarray:
    """zeros, ones on the sub-diagonal, alpha at (1, ell)."""
    C = np.eye(ell, k=-1)
    C[0, ell - 1] = alpha
    return C


def dense_P_alpha(A: np.ndarray, ell: int, alpha: float) -> np.ndarray:
    """P_alpha = I_ell (x) A + C_alpha (x) (-I_N)."""
    N = A.shape[0]
    return np.kron(np.eye(ell), A) - np.kron(C_alpha(ell, alpha), np.eye(N))


def forward(r, ell: int, alpha: float) -> np.ndarray:
    """hat w = (U^* Gamma_alpha (x) I_N) r: gamma-scale each block, then the unitary
    DFT across blocks (numpy FFT, norm='ortho' = ell^{-1/2} sum_j e^{-2 pi i jk/ell})."""
    r = np.asarray(r, dtype=np.float64)
    g = gammas(ell, alpha).reshape((ell,) + (1,) * (r.ndim - 1))
    return np.fft.fft(g * r, axis=0, norm="ortho")


def inverse(yhat, ell: int, alpha: float, imag_tol: float = 1e-10) -> np.ndarray:
    """z = (Gamma_alpha^{-1} U (x) I_N) yhat; the imaginary residue is discarded after
    checking ||Im z|| <= imag_tol ||Re z|| (reading R17)."""
    u = np.fft.ifft(yhat, axis=0, norm="ortho")
    g = gammas(ell, alpha).reshape((ell,) + (1,) * (u.ndim - 1))
    z = u / g
    nr = np.linalg.norm(z.real)
    if nr > 0 and np.linalg.norm(z.imag) > imag_tol * nr:
        raise AssertionError("inverse DFT left an imaginary residue "
                             f"{np.linalg.norm(z.imag) / nr:.3e}")
    return z.real.copy()


def exact_apply(w: op.Weights, r, ell: int, alpha: float) -> np.ndarray:
    """P_alpha^{-1} r by Eq. (eq:Paform) with exact sparse complex solves of
    (A - Lambda_k I) yhat_k = hat w_k for every k (Eq. eq:blockproblem)."""
    r = np.asarray(r).reshape((ell,) + w.shape)
    what = forward(r, ell, alpha)
    A = op.sparse_A(w).astype(np.complex128)
    lam = shifts(ell, alpha)
    yhat = np.empty_like(what)
    I = sp.identity(w.N, dtype=np.complex128, format="csc")
    for k in range(ell):
        yhat[k] = spla.spsolve((A - lam[k] * I).tocsc(), what[k].reshape(-1)).reshape(w.shape)
    return inverse(yhat, ell, alpha)


def smw_inverse(A: np.ndarray, ell: int, alpha: float) -> np.ndarray:
    """Lemma lemma:Zalpha:
    P^{-1} = calA^{-1} + calA^{-1} E_1 Z^{-1} E_ell^T calA^{-1}, Z = alpha^{-1}(I - alpha A^{-ell})."""
    N = A.shape[0]
    calA = op.dense_allatonce(A, ell)
    Ainv = np.linalg.inv(calA)
    E1 = np.zeros((ell * N, N)); E1[:N] = np.eye(N)
    El = np.zeros((ell * N, N)); El[-N:] = np.eye(N)
    Aml = np.linalg.matrix_power(np.linalg.inv(A), ell)
    Z = (np.eye(N) - alpha * Aml) / alpha
    return Ainv + Ainv @ E1 @ np.linalg.inv(Z) @ El.T @ Ainv


def gamma_condition(ell: int, alpha: float) -> float:
    """kappa_2(U^* Gamma_alpha) = max gamma / min gamma (Fig. 2 right)."""
    g = gammas(ell, alpha)
    return float(g.max() / g.min())
