"""Data parallel on real GPUs (NCCL over NVLink): N ranks through the C ABI against the fp64 oracle
on the concatenated rows (S:405 serial equivalence), with bitwise replica consistency (every
worker applies the identical update).  Skipped unless >= 2 GPUs are visible."""
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import mlstm_oracle as O
from synth import bytestream

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("world,plan", [(2, ""), (2, "pair")] + ([(4, "")] if NGPU >= 4 else []))
def test_dp_matches_oracle_on_concatenated_rows(tmp_path, world, plan):
    """plan="pair" forces CTA-pair tiles, so dW_h runs in two row halves whose allreduces start
    while the rest of the weight gradients compute (the C3/C5 bucket schedule)."""
    h, e, B, T, steps = 128, 64, 130, 8, 3
    out = str(tmp_path / "dp")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={29600 + world + (7 if plan else 0)}",
           os.path.join(HERE, "dp_worker.py"), out, str(h), str(e), str(B), str(T), str(steps)]
    env = dict(os.environ, MLSTM_FORCE_PLAN=plan) if plan else None
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    R = [np.load(f"{out}.rank{r}.npz") for r in range(world)]
    # replicas: bitwise identical masters and identical global losses on every rank
    for r in range(1, world):
        assert np.array_equal(R[0]["theta"], R[r]["theta"])
        assert np.array_equal(R[0]["losses"], R[r]["losses"])
    # step 0 against the oracle on all B*world rows (global mean loss and gradient)
    theta0 = O.flatten(O.init_params(h, e, 0x5EED))      # the oracle's own init ...
    assert np.array_equal(R[0]["theta0"], theta0.astype(np.float32))  # ... which every rank started from
    by = bytestream.window(np.arange(B * world), 0, T)
    P = O.unflatten(theta0, h, e)
    z = np.zeros((B * world, h))
    loss_sum, g_ref, _, _ = O.loss_and_grads(P, by, z, z)
    loss_ref = loss_sum / (B * world * T)
    assert abs(R[0]["losses"][0] - loss_ref) <= 5e-3 * loss_ref
    G = O.unflatten(R[0]["grads0"].astype(np.float64), h, e)
    for n in O.PARAM_NAMES:
        a, b = G[n].ravel(), g_ref[n].ravel()
        assert float(a @ b / (np.linalg.norm(a) * np.linalg.norm(b))) >= 0.999, n


@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
def test_dp_micro_batches_and_weight_norm_match_oracle(tmp_path):
    """2 ranks, each step as 2 micro-batches (fp32 accumulation, one allreduce) with weight-normalised
    LSTM matrices (dv, dg formed after the allreduce) against the oracle on the concatenated rows."""
    world, h, e, B, T, steps, micro = 2, 128, 64, 128, 8, 2, 64
    out = str(tmp_path / "dpmw")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", "--master-port=29610", os.path.join(HERE, "dp_worker.py"),
           out, str(h), str(e), str(B), str(T), str(steps), str(micro), "1"]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    R = [np.load(f"{out}.rank{r}.npz") for r in range(world)]
    assert np.array_equal(R[0]["theta"], R[1]["theta"])
    theta0 = O.wn_init(h, e, 0x5EED)
    assert np.allclose(R[0]["theta0"], theta0, rtol=2e-7, atol=0)
    by = bytestream.window(np.arange(B * world), 0, T)
    z = np.zeros((B * world, h))
    loss_sum, g_ref, _, _ = O.wn_loss_and_grads(theta0, h, e, by, z, z)
    loss_ref = loss_sum / (B * world * T)
    assert abs(R[0]["losses"][0] - loss_ref) <= 5e-3 * loss_ref
    G, Gg = O.wn_split(R[0]["grads0"].astype(np.float64), h, e)
    Rf, Rg = O.wn_split(g_ref, h, e)
    for n in O.PARAM_NAMES:
        a, b = G[n].ravel(), Rf[n].ravel()
        assert float(a @ b / (np.linalg.norm(a) * np.linalg.norm(b))) >= 0.999, n
    for n in O.WN_NAMES:
        a, b = Gg[n], Rg[n]
        assert float(a @ b / (np.linalg.norm(a) * np.linalg.norm(b))) >= 0.999, n
