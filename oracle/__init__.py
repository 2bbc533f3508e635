"""ORACLE — test infrastructure only.

A plain, slow, fp64 CPU implementation of what the hot path of arXiv 2506.03947
computes, written from PAPER.md (and the readings listed in DESIGN.md §3) BEFORE
any kernel. It shares no code with the CUDA path (paper_2506_03947_b200/):
neither imports the other. Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s cpu_baseline / `--impl reference` legs may import it.

Deliberately different organisation from the GPU path:
  * every one of the ell Fourier blocks is solved separately in complex
    arithmetic (no half-complex packing, no conjugate-symmetry shortcut);
  * the block DFT is numpy's FFT along the block axis (a library primitive);
  * Galerkin coarse operators are formed as sparse products P^T A P;
  * grids are plain ndarray slices.

Modules (each function cites the passage it follows):
  operator   A, the all-at-once matrix, dense/sparse assembly, recurrence
  circulant  Gamma_alpha, the shifts Lambda_k, block DFT, exact P_alpha
  chebyshev  Chebyshev semi-iteration, sigma bound, p*, Algorithm 1, NC apply
  saddle     saddle-point form, MINRES, PCG, multigrid V-cycle, SP apply
  gmres      flexible GMRES with CGS2 (north_star; not in the paper)
  outer      the paper's outer solver: CI on the left-preconditioned system
  paper      the paper's own Dirichlet test operator + Appendix A bounds

Parity status: every function here is pinned by tests/test_oracle_*.py against
values the paper prints, closed forms, dense linear algebra or brute force,
except where a docstring says "parity unpinned".
"""
from . import operator, circulant, chebyshev, saddle, gmres, paper, outer  # noqa: F401
