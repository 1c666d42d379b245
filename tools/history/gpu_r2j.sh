#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for x in 0 8; do
  echo "== MLSTM_RC_EXP=$x" >> gpurun_out/r2k_trace.log
  MLSTM_RC_EXP=$x timeout 300 python tools/trace_recur.py 2>&1 > /tmp/tr.log
  grep -v "^ *[0-9]" /tmp/tr.log | head -14 >> gpurun_out/r2k_trace.log
  grep -A90 "k-blocks" /tmp/tr.log | head -90 | awk '$1<=50' >> gpurun_out/r2k_trace.log
done
