#!/bin/bash
# round 2: full GPU suite + bench lines (per-timestep default and persistent) with the new bench.py
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/r2r_gpu_tests.log 2>&1
echo "gpu tests exit $?" >> gpurun_out/r2r_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2r_smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/r2r_smoke.log
for rc in 0 1; do
  timeout 600 python bench.py --steps 20 --warmup 5 --recurrence $rc >> gpurun_out/r2r_bench.log 2>&1
  echo "recurrence=$rc exit $?" >> gpurun_out/r2r_bench.log
done
