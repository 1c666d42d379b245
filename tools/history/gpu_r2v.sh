#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_recur.py tests/test_gpu_fullsize.py -q -k "recur or persistent or 4096-256-6-1" > gpurun_out/r2w_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/r2w_tests.log
timeout 300 python tools/trace_recur.py > /tmp/tr.log 2>&1
grep -v "^ *[0-9]" /tmp/tr.log > gpurun_out/r2w_trace.log
for rc in 1 0 1; do
  timeout 600 python bench.py --steps 20 --warmup 5 --recurrence $rc --no-cpu-baseline --no-e2e >> gpurun_out/r2w_bench.log 2>&1
done
