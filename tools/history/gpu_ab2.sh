#!/bin/bash
# parity + A/B of an env knob: bash tools/gpu_ab2.sh VAR
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
V=${1:-MLSTM_ASYNC_EPI}
{
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for x in ${2:-1 0 1 0}; do
  echo "== $V=$x"
  env $V=$x timeout 300 python tools/trace_step.py 2>&1 | grep -E "^(F1|F2|B1|B2) "
  env $V=$x timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e | python3 -c "
import sys,json; d=json.loads(sys.stdin.read()); print('bench', round(d['value']), d['phases_ms_per_step']['fwd_rec'], d['phases_ms_per_step']['bwd_rec'], d['clocks'])"
done
} > gpurun_out/ab2.log 2>&1
cat gpurun_out/ab2.log
