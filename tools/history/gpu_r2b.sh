#!/bin/bash
# round 2: persistent recurrence producer (parallel flag acquire) + per-timestep trace; ABI tests
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_recur.py tests/test_gpu_abi.py -x -q > gpurun_out/r2b_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/r2b_tests.log
for fl in 1 5; do
  echo "== MLSTM_RC_FLAG_LANES=$fl" >> gpurun_out/r2b_trace.log
  MLSTM_RC_FLAG_LANES=$fl timeout 300 python tools/trace_recur.py >> gpurun_out/r2b_trace.log 2>&1
done
for fl in 1 5; do
  MLSTM_RC_FLAG_LANES=$fl timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/r2b_bench.log 2>&1
  echo "flag_lanes=$fl exit $?" >> gpurun_out/r2b_bench.log
done
