#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
{
for v in base NOZS NOLD NOST; do
  echo "== $v"
  if [ $v = base ]; then L=""; else L="MLSTM_LIB=$PWD/paper_1808_01371_b200/libmlstm_$v.so"; fi
  env $L timeout 300 python tools/trace_step.py 2>&1 | grep -E "B2 split|^B2 "
done
} > gpurun_out/abl.log 2>&1
cat gpurun_out/abl.log
