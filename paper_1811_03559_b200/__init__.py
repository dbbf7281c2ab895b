"""paper_1811_03559_b200 — B200-native (sm_100a) recursive SPIKE banded solver.

Drop-in for the reference's C++ solver API (arXiv 1811.03559 artifact,
``proj/include/spike``): factorize / solve / transpose_solve, non-pivoting
(diagonal boosting) and partial-pivoting variants, arbitrary partition counts.
The compute path is hand-written CUDA behind the C-ABI in
``include/spike_b200.h``; this package is the Python mirror of the reference
interface.
"""
from .spike import *  # noqa: F401,F403
from .spike import lib, LIB_PATH  # noqa: F401

__all__ = [n for n in dir() if not n.startswith("_")]
