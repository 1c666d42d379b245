#!/bin/bash
# dW_h side-stream chunks (MLSTM_WGRAD_SIDE): parity tests, then interleaved C3 A/B bench lines
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/side2; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_wgrad_side.py -q -m gpu > $O/tests.log 2>&1
echo "tests exit $?" >> $O/tests.log
for rep in 1 2; do
  for side in none 3,32,10,1 3,32,10,0 2,32,8,1 3,32,6,1 2,32,10,1; do
    if [ $side = none ]; then unset MLSTM_WGRAD_SIDE; else export MLSTM_WGRAD_SIDE=$side; fi
    timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_${side}_$rep.log 2>&1
    echo "exit $?" >> $O/bench_${side}_$rep.log
  done
done
unset MLSTM_WGRAD_SIDE
