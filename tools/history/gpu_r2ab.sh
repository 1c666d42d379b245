#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_recur.py -q > gpurun_out/r2ab_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/r2ab_tests.log
for rc in 0 3 1 0 3 1; do
  timeout 600 python bench.py --steps 20 --warmup 5 --recurrence $rc --no-cpu-baseline --no-e2e > /tmp/b.log 2>&1
  echo "rc=$rc $(grep -o '"value": [0-9.]*' /tmp/b.log | head -1) $(grep -o '"fwd_rec": [0-9.]*' /tmp/b.log | tail -1) $(grep -o '"bwd_rec": [0-9.]*' /tmp/b.log | tail -1) $(grep -o '"optimizer": [0-9.]*' /tmp/b.log | tail -1) $(grep -o '"sm_mhz": [0-9.]*' /tmp/b.log)" >> gpurun_out/r2ab_bench.log
done
