#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for x in 32 48; do
  echo "== MLSTM_RC_EXP=$x" >> gpurun_out/r2o_trace.log
  MLSTM_RC_EXP=$x timeout 300 python tools/trace_recur.py 2>&1 > /tmp/tr.log
  grep -v "^ *[0-9]" /tmp/tr.log | head -14 >> gpurun_out/r2o_trace.log
  grep -A90 "k-blocks" /tmp/tr.log | head -90 | awk '$1>=28 && $1<=40' >> gpurun_out/r2o_trace.log
done
