"""B200-native ProbeSDF fused render + train hot path (arXiv 2412.10084).

The product is ``lib/libpsdf.so`` (C ABI: include/psdf.h) — hand-written
sm_100a kernels for the fused ray pass and the grid update.  ``api`` mirrors
the reference's host API (include/sdfrecon/*.hpp) over that ABI.
"""
from . import _lib  # noqa: F401

__all__ = ["api"]
