#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
{
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "forced or multi_step or micro" 2>&1 | tail -15
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x 2>&1 | tail -15
} > gpurun_out/run9.log 2>&1
cat gpurun_out/run9.log
