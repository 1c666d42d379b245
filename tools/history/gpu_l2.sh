#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
{
timeout 120 python tools/diag_step.py mixed 1024 64 256 16 || echo "DIAG FAILED rc=$?"
for wh in 0.0 0.3 0.5 0.7; do for wmh in 0.0 1.0; do
  echo "WH=$wh WMH=$wmh"; MLSTM_L2_WH=$wh MLSTM_L2_WMH=$wmh timeout 600 python bench.py --steps 5 --warmup 2 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['phases_ms_per_step'], d['clocks'])"
done; done
} > gpurun_out/l2.log 2>&1
cat gpurun_out/l2.log
