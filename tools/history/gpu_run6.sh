#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
{
timeout 120 python tools/diag_step.py mixed 1024 64 256 16 || echo "DIAG FAILED rc=$?"
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
timeout 600 python tools/trace_step.py 2>&1 | grep -v Warn | grep -v nanmean
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('PDL on', d['value'], d['phases_ms_per_step'], d['clocks'])"
MLSTM_PDL=0 timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('PDL off', d['value'], d['phases_ms_per_step'], d['clocks'])"
} > gpurun_out/run6.log 2>&1
tail -30 gpurun_out/run6.log
