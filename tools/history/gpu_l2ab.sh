#!/bin/bash
# L2 residency of the recurrent weights under the power cap: interleaved C3 A/B with board power
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/l2ab; mkdir -p $O
for rep in 1 2 3; do
  for v in base wh05 wh08 wmh1; do
    unset MLSTM_L2_WH MLSTM_L2_WMH
    case $v in wh05) export MLSTM_L2_WH=0.5;; wh08) export MLSTM_L2_WH=0.8;; wmh1) export MLSTM_L2_WMH=1.0;; esac
    timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > $O/bench_${v}_$rep.log 2>&1
    echo "exit $?" >> $O/bench_${v}_$rep.log
  done
done
