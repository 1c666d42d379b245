"""Runs a few C3 train steps (for ncu captures of single kernels): python tools/one_step.py [steps]"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1808_01371_b200 as M  # noqa: E402
from synth import bytestream  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = M.mlstm_default_config(hidden=4096, embed=64, batch=256, seq_len=256)
m = M.MLSTM(cfg)
by = torch.from_numpy(bytestream.window(np.arange(256), 0, 256)).cuda()
for _ in range(steps):
    print(m.train_step(by))
m.close()
