#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
{
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for x in 1 0 1 0; do MLSTM_BWD_PERSIST=$x timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e | python3 -c "
import sys,json; d=json.loads(sys.stdin.read()); p=d['phases_ms_per_step']; print('PERSIST=$x', round(d['value']), 'ms', round(d['ms_per_step'],2), 'fwd', p['fwd_rec'], 'bwd', p['bwd_rec'], d['clocks']['sm_mhz'])"; done
} > gpurun_out/run20.log 2>&1
cat gpurun_out/run20.log
