#!/bin/bash
# round 2: first run of the persistent dataflow recurrence (tests, then an interleaved C3 A/B)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt 2>&1
export MLSTM_RECUR_DEBUG=1
timeout 900 python -m pytest tests/test_gpu_recur.py -x -q > gpurun_out/r2a_recur_tests.log 2>&1
echo "recur tests exit $?" >> gpurun_out/r2a_recur_tests.log
for i in 1 2; do
  MLSTM_RECUR=0 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/r2a_bench.log 2>&1
  echo "A(recur=0) exit $?" >> gpurun_out/r2a_bench.log
  MLSTM_RECUR=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/r2a_bench.log 2>&1
  echo "B(recur=1) exit $?" >> gpurun_out/r2a_bench.log
done
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/r2a_all_gpu.log 2>&1
echo "all gpu tests exit $?" >> gpurun_out/r2a_all_gpu.log
