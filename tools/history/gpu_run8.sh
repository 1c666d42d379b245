#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
{
timeout 600 python tools/trace_step.py 4096 64 1024 256
timeout 1200 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e
timeout 600 python tools/gemm_vs_cublas.py 2>&1 | tail -30
} > gpurun_out/run8.log 2>&1
cat gpurun_out/run8.log
