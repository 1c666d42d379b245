"""Shared helpers for the GPU parity tests: run the CUDA path through the C ABI and the fp64 oracle
on the same seeded inputs and compare with the north_star tolerances (BASELINE.json):
  fp32 mode : loss relative error <= 1e-5, per-tensor gradient relative L2 error <= 1e-4
  mixed mode: loss relative error <= 5e-3, per-tensor gradient cosine >= 0.999
"""
from __future__ import annotations

import numpy as np

from oracle import mlstm_oracle as O
from synth import bytestream

TOL = {"fp32": {"loss_rel": 1e-5, "grad_rel_l2": 1e-4}, "mixed": {"loss_rel": 5e-3, "grad_cos": 0.999}}


def oracle_theta(h, e, seed=0x5EED, weight_norm=False):
    """The oracle's own initial parameters (flat, canonical): every parity test starts the GPU from
    these (pushed through mlstm_set_params), so no oracle input is ever read back from the GPU."""
    return O.wn_init(h, e, seed) if weight_norm else O.flatten(O.init_params(h, e, seed))


def make_model(h, e, B, T, precision, seed=0x5EED, push_oracle=True, **kw):
    import paper_1808_01371_b200 as M
    cfg = M.mlstm_default_config(hidden=h, embed=e, seq_len=T, batch=B, seed=seed,
                                 precision=M.MLSTM_MIXED if precision == "mixed" else M.MLSTM_FP32, **kw)
    m = M.MLSTM(cfg)
    if push_oracle:
        m.set_params(oracle_theta(h, e, seed, bool(kw.get("weight_norm", 0))))
    return m


def to_dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint8)).cuda()


def inputs(B, T, k=0, seed=0x5EED, kind="markov"):
    return bytestream.window(np.arange(B), k, T, seed=seed, kind=kind)


def split(flat, h, e):
    return O.unflatten(np.asarray(flat, dtype=np.float64), h, e)


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def cosine(a, b):
    a, b = a.ravel(), b.ravel()
    na, nb = np.linalg.norm(a), np.linalg.norm(b)
    if na == 0 and nb == 0:
        return 1.0
    return float(a @ b / (na * nb))


def compare_grads(g_gpu, g_ref, h, e, precision):
    G, R = split(g_gpu, h, e), split(g_ref, h, e)
    report = {}
    for n in O.PARAM_NAMES:
        if precision == "fp32":
            report[n] = rel_l2(G[n], R[n])
        else:
            report[n] = cosine(G[n], R[n])
    return report


def oracle_step(params_flat, by, h, e, h0=None, c0=None, alpha=65536.0):
    P = split(params_flat, h, e)
    B = by.shape[0]
    z = np.zeros((B, h))
    loss_sum, g, state, cache = O.loss_and_grads(P, by, z if h0 is None else h0, z if c0 is None else c0,
                                                 scale=1.0)
    return loss_sum / (B * (by.shape[1] - 1)), O.flatten(g), state, cache
