"""Our tcgen05 engines vs cuBLAS (torch.matmul, fp16, fp32 accumulate) on the step's GEMM shapes,
random operands, same process."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import paper_1808_01371_b200 as M
torch.backends.cuda.matmul.allow_fp16_reduced_precision_reduction = False
shapes = [("F2", 256, 16384, 4096), ("F1/B2", 256, 4096, 4096), ("B1", 256, 4096, 16384),
          ("dW_h", 16384, 4096, 65536), ("dW_mh", 4096, 4096, 65536), ("sq8192", 8192, 8192, 8192),
          ("F2@1k", 1024, 16384, 4096), ("F1@1k", 1024, 4096, 4096), ("B1@1k", 1024, 4096, 16384)]
for name, m, n, k in shapes:
    it = 3 if m * n * k > 1e12 else 20
    ours = M.mlstm_gemm_bench(3, m, n, k, 0, it)
    a = torch.randn(m, k, device="cuda", dtype=torch.float16)
    b = torch.randn(n, k, device="cuda", dtype=torch.float16)
    for _ in range(2):
        c = a @ b.T
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(it):
        c = a @ b.T
    e1.record(); torch.cuda.synchronize()
    cub = e0.elapsed_time(e1) / it
    f = 2 * m * n * k / 1e9
    print(f"{name:7s} {m}x{n}x{k}: ours {ours*1e3:8.1f} us {f/ours:7.1f} TF/s | cuBLAS {cub*1e3:8.1f} us {f/cub:7.1f} TF/s", flush=True)
    del a, b, c
