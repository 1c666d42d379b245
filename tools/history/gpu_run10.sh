#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
{
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "forced and not split" 2>&1 | tail -5
MLSTM_FORCE_PLAN=split timeout 900 /usr/local/cuda/bin/compute-sanitizer --print-limit 5 python -m pytest tests/test_gpu_parity.py -q -x -k "forced and split and 256" 2>&1 | grep -v "^=====\s*$" | head -60
} > gpurun_out/run10.log 2>&1
cat gpurun_out/run10.log
