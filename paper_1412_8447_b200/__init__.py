"""B200-native ID / CUR hot path of arXiv 1412.8447 (drop-in for the
reference ``lowrank`` library's randomized / deterministic ID and CUR).

The compute path is liblowrank_b200.so (hand-written sm_100a kernels behind
the C ABI in include/lowrank_b200.h); this package is the Python mirror of
the reference's C++ entry points.
"""
from . import _lib  # noqa: F401
from .lowrank import *  # noqa: F401,F403
from .lowrank import __all__ as _all

__all__ = list(_all)
__version__ = "0.1.0"
