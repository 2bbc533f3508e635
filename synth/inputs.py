"""Seeded problem data for the BASELINE.json configs (no method arithmetic).

Recipe:
  * cell-centred grid, n_a cells per axis, h_a = 1/n_a, x fastest in memory;
  * g(x) = sum_j a_j sin(2*pi*(p_j x + q_j y + r_j z) + phi_j) with M modes
    (M = 4 / 8 / 12 for 1D / 2D / 3D), a_j ~ N(0,1)/M, integer wavenumbers
    uniform in [1, 4], phi_j ~ U[0, 2*pi);
  * kappa = exp(0.5 g) evaluated at the midpoint of every INTERIOR face
    (boundary faces carry no flux under Neumann BCs, so they are not drawn);
    per-axis anisotropy multipliers (the headline uses kappa_y = 0.25 kappa);
  * draws from numpy.random.default_rng(seed) (PCG64) in the order
    a, p, q (2D/3D), r (3D), phi, then b_1 ~ N(0,1) over the N cells in
    C order; blocks 2..ell of b are zero (PAPER.md:43-45 Eq. eq:A).
  * c = L^2 / (2 ell) with L = Lmult * h_x (BASELINE.json:configs).

Face arrays are returned in their natural interior layout:
  kx[nz][ny][nx-1]  face between cells (i, j, k) and (i+1, j, k)
  ky[nz][ny-1][nx]  face between cells (i, j, k) and (i, j+1, k)
  kz[nz-1][ny][nx]  face between cells (i, j, k) and (i, j, k+1)
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np


@dataclasses.dataclass(frozen=True)
class ConfigSpec:
    name: str
    dim: int
    n: int
    ell: int
    alpha: float
    lmult: float          # L = lmult * h
    modes: int
    aniso: tuple          # multiplier per axis (x, y, z)
    method: str           # "nc1" | "nc2" | "sp"
    k: int                # inner iteration budget per shifted system
    rtol: float = 1e-10


CONFIGS = {
    # BASELINE.json configs[0]
    "1d": ConfigSpec("1d", 1, 128, 4, 1e-2, 8.0, 4, (1.0, 1.0, 1.0), "nc1", 10),
    # BASELINE.json configs[1] (alpha in {1e-2, 1e-4}, k in {5, 20})
    "2d256": ConfigSpec("2d256", 2, 256, 10, 1e-2, 10.0, 8, (1.0, 1.0, 1.0), "nc1", 5),
    # BASELINE.json configs[2] -- the headline
    "headline": ConfigSpec("headline", 2, 1024, 10, 1e-4, 10.0, 8, (1.0, 0.25, 1.0), "nc2", 8),
    # BASELINE.json configs[3] -- saddle-point inner solver on the headline operator
    "saddle": ConfigSpec("saddle", 2, 1024, 10, 1e-4, 10.0, 8, (1.0, 0.25, 1.0), "sp", 8),
    # BASELINE.json configs[4]
    "3d": ConfigSpec("3d", 3, 256, 12, 1e-4, 6.0, 12, (1.0, 1.0, 1.0), "nc1", 10),
}


def config(name: str) -> ConfigSpec:
    return CONFIGS[name]


@dataclasses.dataclass
class Problem:
    dim: int
    shape: tuple              # (nz, ny, nx); unused axes are 1
    ell: int
    alpha: float
    c: float                  # diffusion coefficient L^2/(2 ell)
    kx: np.ndarray
    ky: np.ndarray
    kz: np.ndarray
    b: np.ndarray             # [ell][nz][ny][nx] float64
    method: str
    k: int
    rtol: float
    name: str = ""
    seed: int = 0
    bd: tuple = (0.0, 0.0, 0.0)   # Dirichlet boundary-face weights (paper mode), else Neumann
    mu_bounds: tuple = None       # exact spectral bounds of A when known (paper mode)

    @property
    def N(self) -> int:
        nz, ny, nx = self.shape
        return nz * ny * nx


def _field(dim, a, p, q, r, phi, X, Y, Z):
    g = np.zeros(np.broadcast(X, Y, Z).shape)
    for j in range(len(a)):
        arg = 2.0 * math.pi * p[j] * X + phi[j]
        if dim >= 2:
            arg = arg + 2.0 * math.pi * q[j] * Y
        if dim >= 3:
            arg = arg + 2.0 * math.pi * r[j] * Z
        g = g + a[j] * np.sin(arg)
    return np.exp(0.5 * g)


def make_problem(name: str = "headline", *, n=None, shape=None, seed: int = 0,
                 alpha=None, ell=None, k=None, method=None, c=None,
                 rhs: str = "b1") -> Problem:
    """Draw the seeded problem for preset `name`.

    `n` overrides the cells per axis (square/cubic grid); `shape` = (nz, ny, nx)
    overrides it with a non-square grid (tests use ragged sizes such as 37x53).
    `rhs` = "b1" gives b = (b_1, 0, ..., 0); "all" draws every block.
    """
    spec = CONFIGS[name]
    dim = spec.dim
    if shape is None:
        nn = spec.n if n is None else n
        shape = {1: (1, 1, nn), 2: (1, nn, nn), 3: (nn, nn, nn)}[dim]
    nz, ny, nx = shape
    ell = spec.ell if ell is None else ell
    alpha = spec.alpha if alpha is None else alpha
    rng = np.random.default_rng(seed)
    M = spec.modes
    a = rng.standard_normal(M) / M
    p = rng.integers(1, 5, M)
    q = rng.integers(1, 5, M) if dim >= 2 else np.zeros(M, dtype=np.int64)
    r = rng.integers(1, 5, M) if dim >= 3 else np.zeros(M, dtype=np.int64)
    phi = rng.uniform(0.0, 2.0 * math.pi, M)
    N = nx * ny * nz
    b = np.zeros((ell, nz, ny, nx))
    if rhs == "b1":
        b[0] = rng.standard_normal(N).reshape(nz, ny, nx)
    elif rhs == "all":
        b[:] = rng.standard_normal(ell * N).reshape(ell, nz, ny, nx)
    else:
        raise ValueError(rhs)

    hx, hy, hz = 1.0 / nx, 1.0 / ny, 1.0 / nz
    ic = (np.arange(nx) + 0.5) * hx
    jc = (np.arange(ny) + 0.5) * hy
    kc = (np.arange(nz) + 0.5) * hz
    # x-faces at x = i*hx, i = 1..nx-1
    Zc, Yc, Xf = np.meshgrid(kc, jc, np.arange(1, nx) * hx, indexing="ij")
    kx = spec.aniso[0] * _field(dim, a, p, q, r, phi, Xf, Yc, Zc)
    Zc, Yf, Xc = np.meshgrid(kc, np.arange(1, ny) * hy, ic, indexing="ij")
    ky = spec.aniso[1] * _field(dim, a, p, q, r, phi, Xc, Yf, Zc)
    Zf, Yc, Xc = np.meshgrid(np.arange(1, nz) * hz, jc, ic, indexing="ij")
    kz = spec.aniso[2] * _field(dim, a, p, q, r, phi, Xc, Yc, Zf)
    if c is None:
        L = spec.lmult * hx
        c = L * L / (2.0 * ell)
    return Problem(dim=dim, shape=(nz, ny, nx), ell=ell, alpha=alpha, c=float(c),
                   kx=np.ascontiguousarray(kx), ky=np.ascontiguousarray(ky),
                   kz=np.ascontiguousarray(kz), b=b,
                   method=spec.method if method is None else method,
                   k=spec.k if k is None else k, rtol=spec.rtol, name=name, seed=seed)


def make_paper_problem(nx: int, ell: int = 10, alpha: float = 0.01, *, D: float = 0.2,
                       seed: int = 0, method: str = "nc2", eta: float = 0.2) -> Problem:
    """The paper's own test problem (§5): A = I - (nu/h^2) L,
    2D Dirichlet 5-point Laplacian on the n_x x n_x interior vertices, h = 1/(n_x+1),
    nu = D^2/(2 ell - 4), D = 0.2; b = (b_1, 0, ..., 0), b_1 ~ N(0,1) (seeded); inner budget
    ell n_x eta per preconditioner apply (k = n_x eta per block). In face-weight form every
    interior and boundary face carries nu/h^2: kappa = nu (n_x+1)^2 / n_x^2 with c = 1 (the
    library's w_f = c kappa n^2), boundary weights bd = nu/h^2. mu_bounds: Appendix A
    (PAPER.md:998-1020), mu = 1 + (4 nu/h^2)(sin^2(i pi/(2(n_x+1))) + sin^2(j pi/(2(n_x+1)))).
    """
    nu = D * D / (2.0 * ell - 4.0)
    f = nu * (nx + 1) ** 2
    kap = f / float(nx * nx)
    s1 = math.sin(math.pi / (2 * (nx + 1))) ** 2
    sn = math.sin(nx * math.pi / (2 * (nx + 1))) ** 2
    mu_min, mu_max = 1.0 + 4.0 * f * 2 * s1, 1.0 + 4.0 * f * 2 * sn
    rng = np.random.default_rng(seed)
    b = np.zeros((ell, 1, nx, nx))
    b[0] = rng.standard_normal(nx * nx).reshape(1, nx, nx)
    return Problem(dim=2, shape=(1, nx, nx), ell=ell, alpha=alpha, c=1.0,
                   kx=np.full((1, nx, nx - 1), kap), ky=np.full((1, nx - 1, nx), kap),
                   kz=np.zeros((0, nx, nx)), b=b, method=method, k=max(1, round(nx * eta)),
                   rtol=1e-6, name=f"paper{nx}", seed=seed, bd=(f, f, 0.0),
                   mu_bounds=(mu_min, mu_max))


@dataclasses.dataclass
class VaryingProblem(Problem):
    """Problem with varying diagonal blocks: block j has its own
    diffusivity kx_blocks[j] (same layouts as kx); kx/ky/kz hold block 0's."""
    kx_blocks: list = None
    ky_blocks: list = None
    kz_blocks: list = None


def make_varying_problem(name: str = "headline", *, drift: float = 0.5, seed: int = 0, **kw) -> VaryingProblem:
    """Time-varying diffusivity for the varying-block extension (DESIGN.md input recipe): the
    seeded field of `name` (make_problem, same draws) modulated per block j by a second seeded
    random Fourier field g2 of the same recipe (numpy default_rng(seed + 1)):
        kappa_j = kappa * exp(0.5 * drift * (t_j - 1/2) * g2),  t_j = j / (ell - 1),
    so the blocks drift smoothly across the window (drift = 0: every block equals block 0).
    No method arithmetic: face values of seeded fields only."""
    base = make_problem(name, seed=seed, **kw)
    spec = CONFIGS[name]
    dim = base.dim
    nz, ny, nx = base.shape
    ell = base.ell
    rng = np.random.default_rng(seed + 1)
    M = spec.modes
    a = rng.standard_normal(M) / M
    p = rng.integers(1, 5, M)
    q = rng.integers(1, 5, M) if dim >= 2 else np.zeros(M, dtype=np.int64)
    r = rng.integers(1, 5, M) if dim >= 3 else np.zeros(M, dtype=np.int64)
    phi = rng.uniform(0.0, 2.0 * math.pi, M)
    hx, hy, hz = 1.0 / nx, 1.0 / ny, 1.0 / nz
    ic = (np.arange(nx) + 0.5) * hx
    jc = (np.arange(ny) + 0.5) * hy
    kc = (np.arange(nz) + 0.5) * hz
    Zc, Yc, Xf = np.meshgrid(kc, jc, np.arange(1, nx) * hx, indexing="ij")
    ex = _field(dim, a, p, q, r, phi, Xf, Yc, Zc)          # exp(g2 / 2) on x-faces
    Zc, Yf, Xc = np.meshgrid(kc, np.arange(1, ny) * hy, ic, indexing="ij")
    ey = _field(dim, a, p, q, r, phi, Xc, Yf, Zc)
    Zf, Yc, Xc = np.meshgrid(np.arange(1, nz) * hz, jc, ic, indexing="ij")
    ez = _field(dim, a, p, q, r, phi, Xc, Yc, Zf)
    kxb, kyb, kzb = [], [], []
    for j in range(ell):
        s = drift * ((j / (ell - 1) if ell > 1 else 0.0) - 0.5)
        kxb.append(np.ascontiguousarray(base.kx * ex ** s))
        kyb.append(np.ascontiguousarray(base.ky * ey ** s))
        kzb.append(np.ascontiguousarray(base.kz * ez ** s))
    fields = {f.name: getattr(base, f.name) for f in dataclasses.fields(Problem)}
    fields.update(kx=kxb[0], ky=kyb[0], kz=kzb[0], name=base.name + "-varying")
    return VaryingProblem(**fields, kx_blocks=kxb, ky_blocks=kyb, kz_blocks=kzb)
