#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for v in 0 1; do
  echo "== MLSTM_RC_WNORMAL=$v" >> gpurun_out/r2t_trace.log
  if [ $v = 1 ]; then export MLSTM_RC_WNORMAL=1; fi
  timeout 300 python tools/trace_recur.py > /tmp/tr.log 2>&1
  grep -v "^ *[0-9]" /tmp/tr.log | head -14 >> gpurun_out/r2t_trace.log
  grep -A90 "k-blocks" /tmp/tr.log | head -90 | awk '$1>=30 && $1<=40' >> gpurun_out/r2t_trace.log
done
