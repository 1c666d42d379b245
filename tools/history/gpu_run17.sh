#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
{
echo "== C5 trace"; MLSTM_PDL=0 timeout 600 python tools/trace_step.py 8192 64 128 256 2>&1 | tail -12
echo "== C4 trace"; MLSTM_PDL=0 timeout 600 python tools/trace_step.py 4096 64 1024 256 2>&1 | tail -12
echo "== C5 bench"; timeout 900 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | python3 -c "
import sys,json; d=json.loads(sys.stdin.read()); print('C5', round(d['value']), d['phases_ms_per_step'], d['clocks'])"
} > gpurun_out/run17.log 2>&1
cat gpurun_out/run17.log
