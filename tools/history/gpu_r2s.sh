#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -k "not dp" > gpurun_out/r2s_gpu_tests.log 2>&1
echo "gpu tests exit $?" >> gpurun_out/r2s_gpu_tests.log
