#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
{
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "forced and persist" 2>&1 | tail -4
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 600 python tools/trace_step.py 2>&1 | tail -12
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e | python3 -c "
import sys,json; d=json.loads(sys.stdin.read()); print('C3 bench', round(d['value']), d['phases_ms_per_step'], d['clocks'])"
timeout 1200 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e | python3 -c "
import sys,json; d=json.loads(sys.stdin.read()); print('C4 bench', round(d['value']), d['phases_ms_per_step'], d['clocks'])"
} > gpurun_out/run14.log 2>&1
cat gpurun_out/run14.log
