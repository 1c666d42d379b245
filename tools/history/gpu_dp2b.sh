#!/bin/bash
# 2 GPUs: DP parity tests, then the C3 and C5 benches with the overlapped vs post-graph allreduce
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
{
timeout 600 python -m pytest tests/test_gpu_dp.py -q -x 2>&1 | tail -5
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k forced 2>&1 | tail -5
for ov in 1 0 1; do
  echo "== MLSTM_AR_OVERLAP=$ov C3"
  MLSTM_AR_OVERLAP=$ov timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e
done
for ov in 1 0; do
  echo "== MLSTM_AR_OVERLAP=$ov C5"
  MLSTM_AR_OVERLAP=$ov timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --config C5 --gpus 2 --steps 5 --warmup 3 --no-e2e
done
} > gpurun_out/dp2b.log 2>&1
grep -v "^W1\|OMP_NUM\|^\*\*\*" gpurun_out/dp2b.log | python3 -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print('value', round(d['value']), 'ms', round(d['ms_per_step'],2), 'phases', d.get('phases_ms_per_step'), 'clk', d.get('clocks'))
    else: print(l.rstrip()[:300])
"
