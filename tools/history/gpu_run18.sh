#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
{
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "forced" 2>&1 | tail -3
timeout 600 python tools/gemm512.py
for x in 0 1 0 1; do MLSTM_WGRAD512=$x timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e | python3 -c "
import sys,json; d=json.loads(sys.stdin.read()); p=d['phases_ms_per_step']; print('W512=$x', round(d['value']), 'wgrad', p['wgrad'], d['clocks']['sm_mhz'])"; done
} > gpurun_out/run18.log 2>&1
cat gpurun_out/run18.log
