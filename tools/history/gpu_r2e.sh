#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 300 python tools/trace_recur.py > gpurun_out/r2e_trace.log 2>&1
