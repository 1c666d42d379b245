import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_1808_01371_b200 as M
eng, m, n, k, bn = map(int, sys.argv[1:6])
ms = M.mlstm_gemm_bench(eng, m, n, k, bn, 2)
print(f"engine={eng} {m}x{n}x{k} bn={bn}: {ms*1e3:.1f} us {2*m*n*k/ms/1e9:.1f} TFLOP/s")
