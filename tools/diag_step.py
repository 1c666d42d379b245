"""Diagnostic: one train step of a small config through the C ABI vs the fp64 oracle.
usage: python tools/diag_step.py precision h e B T   (MLSTM_DEBUG_SIMT_GEMM=1 forces the SIMT engine)"""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
from gpu_helpers import make_model, inputs, oracle_step, compare_grads, to_dev

prec = sys.argv[1]; h, e, B, T = map(int, sys.argv[2:6])
t0 = time.time()
m = make_model(h, e, B, T, prec)
theta0 = m.get_params().astype(np.float64)
by = inputs(B, T)
r = m.train_step(to_dev(by))
t1 = time.time()
loss_ref, g_ref, _, _ = oracle_step(theta0, by, h, e)
g = m.get_grads().astype(np.float64)
rep = compare_grads(g, g_ref, h, e, prec)
print(f"{prec} h={h} B={B} T={T} simt={os.environ.get('MLSTM_DEBUG_SIMT_GEMM','0')} loss gpu={r['loss_nats']:.8f} "
      f"ref={loss_ref:.8f} rel={abs(r['loss_nats']-loss_ref)/loss_ref:.2e} skipped={r['skipped']} gpu_s={t1-t0:.1f}")
print("  ", {k: f"{v:.6f}" for k, v in rep.items()})
