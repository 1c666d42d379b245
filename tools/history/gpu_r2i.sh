#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for hh in 1024 2048 4096; do
  echo "== h=$hh" >> gpurun_out/r2i_trace.log
  timeout 300 python tools/trace_recur.py $hh 256 256 2>&1 | grep -v "^ *[0-9]" | head -14 >> gpurun_out/r2i_trace.log
  timeout 300 python tools/trace_recur.py $hh 256 256 2>&1 | grep -A40 "k-blocks" | head -40 >> gpurun_out/r2i_trace.log
done
