#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
{
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -30
timeout 600 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e
timeout 900 python bench.py --steps 10 --warmup 3
} > gpurun_out/run2.log 2>&1
tail -50 gpurun_out/run2.log
