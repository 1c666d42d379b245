#!/bin/bash
# persistent BPTT: K-major transposed weights (one box per stage) vs MN-major (two boxes), interleaved
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
MLSTM_RC_WKM=1 timeout 900 python -m pytest tests/test_gpu_recur.py -q > gpurun_out/r2y_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/r2y_tests.log
for w in 1 0 1 0; do
  MLSTM_RC_WKM=$w timeout 600 python bench.py --steps 20 --warmup 5 --recurrence 1 --no-cpu-baseline --no-e2e > /tmp/b.log 2>&1
  echo "WKM=$w $(grep -o '"value": [0-9.]*' /tmp/b.log | head -1) $(grep -o '"bwd_rec": [0-9.]*' /tmp/b.log | head -1) $(grep -o '"optimizer": [0-9.]*' /tmp/b.log | head -1) $(grep -o '"sm_mhz": [0-9.]*' /tmp/b.log)" >> gpurun_out/r2y_bench.log
done
