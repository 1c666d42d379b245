#!/bin/bash
# round 2: producer learns activation readiness ahead of need (flag window), trace + bench
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_recur.py -x -q > gpurun_out/r2d_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/r2d_tests.log
timeout 300 python tools/trace_recur.py > gpurun_out/r2d_trace.log 2>&1
for i in 1; do
  MLSTM_RECUR=0 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/r2d_bench.log 2>&1
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/r2d_bench.log 2>&1
done
