#!/bin/bash
# round 2: 8192-d tests, C5 (paper LR) and C5-256 bench lines, C4
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -k "8192 or invariance" > gpurun_out/r2u_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/r2u_tests.log
for cfg in C5 C5-256 C4; do
  timeout 900 python bench.py --config $cfg --steps 10 --warmup 5 --no-cpu-baseline >> gpurun_out/r2u_bench.log 2>&1
  echo "$cfg exit $?" >> gpurun_out/r2u_bench.log
done
