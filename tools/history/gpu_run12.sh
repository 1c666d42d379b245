#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
{
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
timeout 600 python tools/trace_step.py 2>&1 | tail -14
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e
} > gpurun_out/run12.log 2>&1
cat gpurun_out/run12.log
