"""Engine throughput sweep: python tools/gemm_sweep.py"""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_1808_01371_b200 as M
shapes = [("F2", 256, 16384, 4096), ("F1/B2", 256, 4096, 4096), ("B1", 256, 4096, 16384),
          ("sq8192", 8192, 8192, 8192), ("dW_mh", 4096, 4096, 65536), ("dW_h", 16384, 4096, 65536)]
for name, m, n, k in shapes:
    it = 3 if m * n * k > 1e12 else 20
    for eng in (1, 2):
        for bn in (64, 128, 256):
            try:
                ms = M.mlstm_gemm_bench(eng, m, n, k, bn, it)
                print(f"{name:7s} M={m:6d} N={n:6d} K={k:6d} engine={eng} bn={bn:3d}: {ms*1e3:9.1f} us "
                      f"{2*m*n*k/ms/1e9:7.1f} TFLOP/s", flush=True)
            except Exception as ex:
                print(name, eng, bn, "ERR", ex, flush=True)
