"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds NO arithmetic of the method (no operator, no transform, no
solver). It only draws the random problem data that `BASELINE.json:configs`
describes (the log-normal diffusivity field sampled at cell faces and the
right-hand side b = (b_1, 0, ..., 0)), so both sides of a parity test see the
identical arrays. make_paper_problem also states the paper's own test problem
in face-weight form, with the spectral bounds the paper's experiments take as given
(Appendix A closed form) -- problem data, like kappa; the oracle pins its own
copy of that formula against dense eigenvalues.
"""
from .inputs import CONFIGS, Problem, VaryingProblem, make_problem, make_paper_problem, make_varying_problem, config  # noqa: F401
