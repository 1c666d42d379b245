"""torchrun worker for tests/test_gpu_dp.py: N ranks train a small mLSTM data-parallel through the
C ABI (NCCL allreduce inside libmlstm) and dump per-rank results."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1808_01371_b200 as M  # noqa: E402
from synth import bytestream  # noqa: E402


def main():
    out, h, e, B, T, steps = sys.argv[1], *map(int, sys.argv[2:7])
    micro = int(sys.argv[7]) if len(sys.argv) > 7 else 0
    wn = int(sys.argv[8]) if len(sys.argv) > 8 else 0
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    t = torch.zeros(128, dtype=torch.uint8, device="cuda")
    if rank == 0:
        t.copy_(torch.frombuffer(bytearray(M.mlstm_nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(t, 0)
    cfg = M.mlstm_default_config(hidden=h, embed=e, batch=B, seq_len=T, precision=M.MLSTM_MIXED,
                                 micro_batch=micro, weight_norm=wn)
    m = M.MLSTM(cfg, rank=rank, world=world, nccl_id=bytes(t.cpu().numpy().tobytes()))
    theta0 = m.get_params()
    rows = np.arange(rank * B, (rank + 1) * B)
    losses, grads0 = [], None
    for k in range(steps):
        by = torch.from_numpy(bytestream.window(rows, k, T)).cuda()
        r = m.train_step(by)
        losses.append(r["loss_nats"])
        if k == 0:
            grads0 = m.get_grads()
    np.savez(f"{out}.rank{rank}.npz", theta0=theta0, theta=m.get_params(), losses=np.array(losses), grads0=grads0)
    m.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
