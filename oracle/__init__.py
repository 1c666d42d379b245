"""fp64 CPU oracle for arXiv 1808.01371's mLSTM training step.

TEST INFRASTRUCTURE ONLY: imported solely by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  Independent of the CUDA path.
"""
from .mlstm_oracle import *  # noqa: F401,F403
from . import mlstm_oracle  # noqa: F401
