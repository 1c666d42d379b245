#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_recur.py tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -k "recur or 4096-256-6-1 or gather" > gpurun_out/r2ac_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/r2ac_tests.log
timeout 300 python tools/trace_recur.py > /tmp/tr.log 2>&1
grep -A30 "^bwd" /tmp/tr.log | grep -v "^ *[0-9]" > gpurun_out/r2ac_trace.log
for rc in 1 0 1 0; do
  timeout 600 python bench.py --steps 20 --warmup 5 --recurrence $rc --no-cpu-baseline --no-e2e > /tmp/b.log 2>&1
  echo "rc=$rc $(grep -o '"value": [0-9.]*' /tmp/b.log | head -1) $(grep -o '"phases_ms_per_step": {[^}]*}' /tmp/b.log) $(grep -o '"sm_mhz": [0-9.]*' /tmp/b.log)" >> gpurun_out/r2ac_bench.log
done
