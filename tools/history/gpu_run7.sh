#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
{
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e | cut -c1-400
timeout 900 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | cut -c1-600
timeout 1200 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e | cut -c1-600
} > gpurun_out/run7.log 2>&1
cat gpurun_out/run7.log
