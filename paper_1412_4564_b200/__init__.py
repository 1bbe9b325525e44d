"""ck -- a B200-native (sm_100a) implementation of MatConvNet's
computational-block hot path (arXiv 1412.4564), behind the reference's block
API.  The compute lives in libck.so (hand-written CUDA + a C ABI, see
include/ck/ck.h); this package is the thin host-side mirror used by callers,
tests and the benchmark.
"""
from ._lib import LIB_PATH, CkError, DataError, ShapeError, lib  # noqa: F401

__all__ = ["lib", "LIB_PATH", "CkError", "ShapeError", "DataError"]
