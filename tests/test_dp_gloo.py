"""Data-parallel host logic on CPU with real torch.distributed ranks (gloo, world_size 2).

The GPU path shards the global batch by rows (rank r owns rows [r*B, (r+1)*B), "distributed
evenly"), seeds dY with alpha/(B_g*T) and SUM-allreduces fp16 gradients (Q7); every rank
then runs the identical overflow check / scaler / Adam (no parameter server).  Here the same
protocol runs with the oracle on each rank and gloo as the collective; it must equal one rank
training on the concatenated rows (S:405 serial equivalence), and replicas must stay identical.
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import mlstm_oracle as O
from synth import bytestream

H, E, B, T, STEPS, WORLD = 8, 64, 3, 5, 3, 2


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    st = O.new_train_state(H, E, B, seed=7)
    rows = np.arange(rank * B, (rank + 1) * B)

    def allreduce(x):
        t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return t.numpy()

    losses = []
    for k in range(STEPS):
        by = bytestream.window(rows, k, T)
        out = O.train_step(st, by, n_global_rows=B * world, grads_hook=allreduce,
                           loss_hook=lambda l: float(allreduce(np.array([l]))[0]))
        losses.append(out["loss_nats"])
    # replica hash: every rank must hold bitwise-identical masters
    digest = torch.tensor([float(np.frombuffer(st.theta.tobytes(), dtype=np.uint64).sum() % (1 << 52))],
                          dtype=torch.float64)
    gathered = [torch.zeros_like(digest) for _ in range(world)]
    dist.all_gather(gathered, digest)
    q.put((rank, st.theta, losses, [g.item() for g in gathered]))
    dist.destroy_process_group()


def test_two_rank_step_equals_one_rank_on_concatenated_rows():
    port = 29500 + (os.getpid() % 1000)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, WORLD, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(WORLD):
        r, theta, losses, digests = q.get(timeout=300)
        res[r] = (theta, losses, digests)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert np.array_equal(res[0][0], res[1][0])               # replicas identical
    assert len(set(res[0][2])) == 1
    # serial reference: one rank, all B*world rows
    st = O.new_train_state(H, E, B * WORLD, seed=7)
    for k in range(STEPS):
        by = bytestream.window(np.arange(B * WORLD), k, T)
        out = O.train_step(st, by)
        assert out["loss_nats"] == pytest.approx(res[0][1][k], rel=1e-12)
    assert np.abs(st.theta - res[0][0]).max() < 1e-12


def test_row_assignment_is_rank_independent():
    """Rank r's rows are exactly rows [rB, (r+1)B) of the 1-rank global batch stream."""
    g = bytestream.window(np.arange(4 * B), 2, T)
    for r in range(4):
        assert np.array_equal(bytestream.window(np.arange(r * B, (r + 1) * B), 2, T), g[r * B:(r + 1) * B])
