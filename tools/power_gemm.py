"""Is the power-capped clock set by operand bytes per FLOP?  Runs the same large GEMM (M=4096, N=16384,
K=4096) for ~6 s on (1) 1-CTA 128x256 tiles (11.4 B of operands per kFLOP) and (2) CTA-pair 256x256 tiles
(7.6 B/kFLOP), sampling board power and SM clock every 100 ms, and reports TFLOP/s, median MHz and W.
Same clock + different speed: issue-bound; lower clock for (1) at the same power: bytes drive power.
python tools/power_gemm.py > gpurun_out/power_gemm.txt"""
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402

import paper_1808_01371_b200 as M  # noqa: E402

Mm, N, K = 4096, 16384, 4096
flop = 2.0 * Mm * N * K
M.mlstm_gemm_bench(1, Mm, N, K, 256, 3)
M.mlstm_gemm_bench(2, Mm, N, K, 256, 3)
for rep in range(2):
    for eng, name in [(1, "1-CTA 128x256 (11.4 B/kFLOP)"), (2, "pair 256x256 (7.6 B/kFLOP)")]:
        p = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw",
                              "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, text=True)
        t0 = time.time()
        ms = []
        while time.time() - t0 < 8.0:
            ms.append(M.mlstm_gemm_bench(eng, Mm, N, K, 256, 2000))
        p.terminate()
        rows = []
        for ln in p.stdout.read().splitlines():
            try:
                a, b = (float(x) for x in ln.split(","))
                rows.append((a, b))
            except ValueError:
                pass
        rows = [r for r in rows[5:] if r[1] > 300]  # drop idle gaps between calls
        sm = np.median([r[0] for r in rows])
        pw = np.median([r[1] for r in rows])
        tf = flop / (np.median(ms[1:]) * 1e-3) / 1e12
        print(f"rep {rep} {name:32s} {tf:7.1f} TFLOP/s  {sm:6.0f} MHz  {pw:6.0f} W  "
              f"{tf * 1e3 / sm:6.3f} TFLOP/s per GHz", flush=True)
