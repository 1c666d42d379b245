#!/bin/bash
# F2 / B1 stream rate without per-block trace records (per-timestep records only)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for x in 64 96 64 96; do
  echo "== MLSTM_RC_EXP=$x" >> gpurun_out/r2z_trace.log
  MLSTM_RC_EXP=$x timeout 300 python tools/trace_recur.py > /tmp/tr.log 2>&1
  grep "^fwd\|^bwd\|F2 Mblk0\|F2 commit\|B1 blk0\|B1 commit\|F1 blk0\|F1 commit\|B2 dAblk0\|B2 commit" /tmp/tr.log >> gpurun_out/r2z_trace.log
done
