"""dW_h-shaped GEMM: CTA-pair tiles 256x256 (non-persistent / persistent) vs 256x512."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_1808_01371_b200 as M
for (m, n, k) in [(16384, 4096, 65536), (4096, 4096, 65536), (16384, 4096, 262144)]:
    f = 2.0 * m * n * k / 1e12
    for eng, bn, name in [(2, 256, "pair256"), (3, 0, "auto(persist)"), (2, 512, "pair512")]:
        ms = M.mlstm_gemm_bench(eng, m, n, k, bn, 3)
        print(f"{m}x{n}x{k} {name:14s} {ms:8.3f} ms {f / ms * 1e3:7.1f} TF/s", flush=True)
