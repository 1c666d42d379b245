#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
{
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 600 python tools/trace_step.py 4096 64 1024 256 2>&1 | grep -E "^(F1|F2|B1|B2) "
timeout 1200 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e | python3 -c "
import sys,json; d=json.loads(sys.stdin.read()); print('C4 bench', round(d['value']), d['phases_ms_per_step'], d['clocks'], d['loss_first_last'])"
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e | python3 -c "
import sys,json; d=json.loads(sys.stdin.read()); print('C3 bench', round(d['value']), d['phases_ms_per_step'], d['clocks'])"
} > gpurun_out/run13.log 2>&1
cat gpurun_out/run13.log
