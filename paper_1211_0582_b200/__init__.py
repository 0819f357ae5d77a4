"""B200-native nodal-DG Maxwell RHS + LSERK4 (arXiv:1211.0582 hot path).

The compute lives in libdg.so (hand-written sm_100a CUDA behind the C ABI of
include/dg.h); `dg` is the ctypes binding.  Importing the package loads the
library and raises if it is missing: there is no CPU fallback.
"""
from . import dg  # noqa: F401
from .dg import Solver, DGError  # noqa: F401

__all__ = ["dg", "Solver", "DGError"]
