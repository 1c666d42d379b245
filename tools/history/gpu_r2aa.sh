#!/bin/bash
# per-timestep backward reading MN-major weights (no transposes): full GPU suite, interleaved bench, launch list
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/r2aa_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/r2aa_tests.log
for i in 1 2; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > /tmp/b.log 2>&1
  echo "$(grep -o '"value": [0-9.]*' /tmp/b.log | head -1) $(grep -o '"phases_ms_per_step": {[^}]*}' /tmp/b.log) $(grep -o '"sm_mhz": [0-9.]*' /tmp/b.log)" >> gpurun_out/r2aa_bench.log
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 1100 -c 1100 --csv \
  --log-file gpurun_out/r2aa_launches.csv python tools/one_step.py 2 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2aa_launches.csv > gpurun_out/r2aa_launch_summary.txt 2>&1
