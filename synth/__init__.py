"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds NO arithmetic of the method (no operator, no transform, no
solver). It only draws the random problem data that `BASELINE.json:configs`
describes (the log-normal diffusivity field sampled at cell faces and the
right-hand side b = (b_1, 0, ..., 0)), so both sides of a parity test see the
identical arrays.
"""
from .inputs import CONFIGS, Problem, make_problem, config  # noqa: F401
