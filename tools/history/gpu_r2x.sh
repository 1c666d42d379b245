#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_abi.py tests/test_gpu_weight_norm.py -q > gpurun_out/r2x_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/r2x_tests.log
for rc in 0 1; do
  timeout 600 python bench.py --steps 20 --warmup 5 --recurrence $rc --no-cpu-baseline --no-e2e >> gpurun_out/r2x_bench.log 2>&1
done
