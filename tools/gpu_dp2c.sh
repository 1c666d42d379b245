#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
N=${1:-2}
{
nvidia-smi -L
timeout 600 python -m pytest tests/test_gpu_dp.py -q -x 2>&1 | tail -3
for cfg in C3 C5; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29531 bench.py --config $cfg --gpus $N --steps 10 --warmup 3 2>&1 | grep "^{" | python3 -c "
import sys,json; d=json.loads(sys.stdin.read()); print('$cfg N=$N', round(d['value']), 'ms', round(d['ms_per_step'],2), d['phases_ms_per_step'], d['clocks'], 'e2e', round(d['e2e']['value']) if d.get('e2e') else None)"
done
} > gpurun_out/dp${N}c.log 2>&1
cat gpurun_out/dp${N}c.log
