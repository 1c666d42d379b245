import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_1808_01371_b200 as M
for name, m, n, k in [("F2", 256, 16384, 4096), ("F1/B2", 256, 4096, 4096), ("B1", 256, 4096, 16384),
                      ("dW_dec", 256, 4096, 65536), ("dHdec", 65536, 4096, 256), ("Y", 65536, 256, 4096)]:
    for eng, bn in ((1, 0), (2, 256), (3, 0)):
        ms = M.mlstm_gemm_bench(eng, m, n, k, bn, 20)
        print(f"{name:7s} M={m:6d} N={n:6d} K={k:6d} engine={eng} bn={bn}: {ms*1e3:9.1f} us {2*m*n*k/ms/1e9:7.1f} TFLOP/s", flush=True)
