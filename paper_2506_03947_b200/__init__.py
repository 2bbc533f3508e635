"""B200-native all-at-once diffusion-covariance solver (arXiv 2506.03947).

The product path is libaac.so (hand-written sm_100a CUDA behind the C ABI of
include/aac.h); `Solver` is its thin ctypes front end. Importing this package
loads libaac.so and raises ImportError if it has not been built.
"""
from .solver import Solver, from_problem, slab_range  # noqa: F401
from ._lib import METHODS, AacError  # noqa: F401

__all__ = ["Solver", "from_problem", "slab_range", "METHODS", "AacError"]
