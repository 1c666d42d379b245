"""C4 validation run: 100 mixed-precision steps at 4096 rows/GPU
(4 x 1024-row micro-batches), h=4096, T=256, lr0=3e-3, D=100k, on the synthetic order-2 Markov stream.
Usage: c4_trace.py [out.json] [steps] [C4|C3|C5] (C3/C5: the same checks at those configs).

Checks: every loss finite, no divergence, 10-step moving average non-increasing (after the first
window), every step's BPC above the source's entropy floor H, skipped steps <= 3.
Writes the per-step trace as JSON (argv[1], default gpurun_out/c4_trace.json)."""
import json, os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np, torch
import paper_1808_01371_b200 as M
from synth import bytestream

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/c4_trace.json"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
cfgname = sys.argv[3] if len(sys.argv) > 3 else "C4"
# C4-32k: SURVEY C4's global batch of 32768 rows (8 GPUs x 4096) on one GPU as 32 micro-batches of
# 1024 rows: the data-parallel SUM over rows is the same arithmetic as one rank's micro-batch sum
h, e, B, T, mb = {"C4": (4096, 64, 4096, 256, 1024), "C4-32k": (4096, 64, 32768, 256, 1024),
                  "C3": (4096, 64, 256, 256, 0), "C5": (8192, 64, 128, 256, 0)}[cfgname]
cfg = M.mlstm_default_config(hidden=h, embed=e, batch=B, seq_len=T, micro_batch=mb, precision=M.MLSTM_MIXED)
m = M.MLSTM(cfg)
floor = bytestream.source().entropy_rate_bits()
t0 = time.time()
data = bytestream.windows(np.arange(B), 0, steps, T)
print(f"generated {data.shape} in {time.time() - t0:.1f}s; entropy floor {floor:.4f} bits", flush=True)
dev = torch.from_numpy(data).cuda()
trace = []
t0 = time.time()
for k in range(steps):
    r = m.train_step(dev[k])
    trace.append({"step": k, "bpc": r["bpc"], "loss_nats": r["loss_nats"], "skipped": int(r["skipped"]),
                  "loss_scale": r["loss_scale"], "lr": r["lr"]})
    if k % 10 == 0 or k == steps - 1:
        print(f"step {k:3d} bpc {r['bpc']:.4f} scale {r['loss_scale']:.0f} skipped {r['skipped']} "
              f"lr {r['lr']:.6g} ({time.time() - t0:.1f}s)", flush=True)
bpc = np.array([t["bpc"] for t in trace])
skips = sum(t["skipped"] for t in trace)
win = 10 if cfgname.startswith("C4") else 25  # smaller batches: noisier per-step BPC, wider moving average
ma = np.convolve(bpc, np.ones(win) / win, mode="valid")
checks = {
    "finite": bool(np.isfinite(bpc).all()),
    "above_floor": bool((bpc > floor).all()),
    "moving_avg_non_increasing": bool((np.diff(ma) <= 1e-3).all()),
    "skipped_le_3": skips <= 3,
    "decreased": bool(bpc[-10:].mean() < bpc[:10].mean()),
}
res = {"config": {"name": cfgname, "hidden": h, "embed": e, "rows_per_gpu": B, "micro_batch": mb, "seq_len": T, "n_gpus": 1,
                  "precision": "mixed", "lr0": 3e-3, "decay_iters": 100000, "data": "synthetic markov order-2"},
       "entropy_floor_bits": floor, "skipped": skips, "checks": checks,
       "wall_s": time.time() - t0, "trace": trace}
os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
json.dump(res, open(out, "w"), indent=1)
print(json.dumps({k: v for k, v in res.items() if k != "trace"}))
assert all(checks.values()), checks
