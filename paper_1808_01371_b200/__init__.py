"""B200-native (sm_100a) mixed-precision, data-parallel mLSTM training step of arXiv 1808.01371.

The compute path lives in libmlstm.so (csrc/, C ABI in include/mlstm.h); this package is the
thin ctypes binding (``mlstm``) and its in-tree build (``build``).
"""
from .mlstm import *  # noqa: F401,F403
from . import mlstm  # noqa: F401
