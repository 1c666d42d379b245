#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
{
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -5
timeout 900 python tools/c4_trace.py gpurun_out/c4_trace.json 100 2>&1 | tail -16
} > gpurun_out/run11.log 2>&1
cat gpurun_out/run11.log
