#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
{
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "train_step_parity and C2" 2>&1 | tail -15
echo "rc=$?"
} > gpurun_out/run19.log 2>&1
cat gpurun_out/run19.log
