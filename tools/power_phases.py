"""Board power and SM clock while the GPU runs (a) only forward recurrences (mlstm_eval, no weight-gradient
GEMMs) and (b) whole C3 training steps, each for ~8 s, sampled by nvidia-smi every 100 ms: does the
recurrence itself run at the power cap, or do the dense weight-gradient phases pull its clock down?
python tools/power_phases.py > gpurun_out/power_phases.txt"""
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1808_01371_b200 as M  # noqa: E402
from synth import bytestream  # noqa: E402


def sample(fn, seconds=8.0):
    p = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap",
                          "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, text=True)
    t0 = time.time()
    n = 0
    while time.time() - t0 < seconds:
        fn()
        n += 1
    torch.cuda.synchronize()
    p.terminate()
    rows = []
    for ln in p.stdout.read().splitlines():
        parts = [x.strip() for x in ln.split(",")]
        try:
            rows.append((float(parts[0]), float(parts[1]), parts[2]))
        except (ValueError, IndexError):
            pass
    rows = rows[5:]  # drop the ramp
    sm = np.array([r[0] for r in rows])
    pw = np.array([r[1] for r in rows])
    cap = sum(r[2].lower().startswith("active") for r in rows)
    return n, sm, pw, cap


cfg = M.mlstm_default_config(hidden=4096, embed=64, batch=256, seq_len=256)
m = M.MLSTM(cfg)
by = torch.from_numpy(bytestream.window(np.arange(256), 0, 256)).cuda()
m.train_step(by)
m.eval(by)
torch.cuda.synchronize()
for name, fn in [("eval (forward recurrence only)", lambda: m.eval(by)), ("train step", lambda: m.train_step(by)),
                 ("eval again", lambda: m.eval(by))]:
    n, sm, pw, cap = sample(fn)
    print(f"{name:32s} calls {n:4d}  sm MHz median {np.median(sm):.0f} (p10 {np.percentile(sm, 10):.0f}, "
          f"p90 {np.percentile(sm, 90):.0f})  power W median {np.median(pw):.0f} (max {pw.max():.0f})  "
          f"sw_power_cap in {cap}/{len(sm)} samples", flush=True)
m.close()
