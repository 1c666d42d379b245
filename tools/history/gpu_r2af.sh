#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for rc in 1 0 1 0 1 0; do
  timeout 600 python bench.py --steps 20 --warmup 5 --recurrence $rc --no-cpu-baseline --no-e2e > /tmp/b.log 2>&1
  echo "rc=$rc $(grep -o '"value": [0-9.]*' /tmp/b.log | head -1) $(grep -o '"phases_ms_per_step": {[^}]*}' /tmp/b.log) $(grep -o '"sm_mhz": [0-9.]*' /tmp/b.log)" >> gpurun_out/r2af_bench.log
done
