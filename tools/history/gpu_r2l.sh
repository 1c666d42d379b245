#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_recur.py -x -q > gpurun_out/r2q_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/r2q_tests.log
timeout 300 python tools/trace_recur.py > /tmp/tr.log 2>&1
grep -v "^ *[0-9]" /tmp/tr.log > gpurun_out/r2q_trace.log
grep -A90 "k-blocks" /tmp/tr.log | head -90 | awk '$1<=50' >> gpurun_out/r2q_trace.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/r2q_bench.log 2>&1
