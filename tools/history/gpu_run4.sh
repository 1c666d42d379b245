#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
{
timeout 300 python tools/gemm_sweep2.py
timeout 120 python tools/diag_step.py mixed 1024 64 256 16 || echo "DIAG FAILED rc=$?"
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -15
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline
} > gpurun_out/run4.log 2>&1
tail -40 gpurun_out/run4.log
