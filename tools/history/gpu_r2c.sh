#!/bin/bash
# round 2: weight L2 prefetch distance sweep of the persistent recurrence, with per-block traces
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
MLSTM_RC_PF=16 timeout 600 python -m pytest tests/test_gpu_recur.py -x -q > gpurun_out/r2c_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/r2c_tests.log
for pf in 0 8 16 32; do
  echo "== MLSTM_RC_PF=$pf" >> gpurun_out/r2c_trace.log
  MLSTM_RC_PF=$pf timeout 300 python tools/trace_recur.py >> gpurun_out/r2c_trace.log 2>&1
done
for pf in 0 16; do
  MLSTM_RC_PF=$pf timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/r2c_bench.log 2>&1
  echo "pf=$pf exit $?" >> gpurun_out/r2c_bench.log
done
