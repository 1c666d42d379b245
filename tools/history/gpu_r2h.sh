#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for x in 0 1 2 3; do
  echo "== MLSTM_RC_EXP=$x" >> gpurun_out/r2h_trace.log
  MLSTM_RC_EXP=$x timeout 300 python tools/trace_recur.py 2>&1 | grep -v "^ *[0-9]" | head -14 >> gpurun_out/r2h_trace.log
done
