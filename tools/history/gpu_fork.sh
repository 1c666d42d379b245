#!/bin/bash
# weight-gradient fork (S GEMM beside dW_h/dW_mh) + side-chunk micro-batch test, interleaved C3 A/B
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/fork; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_wgrad_side.py -q -m gpu > $O/tests.log 2>&1
echo "tests exit $?" >> $O/tests.log
for rep in 1 2 3; do
  for fk in 0 1; do
    MLSTM_WGRAD_FORK=$fk timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > $O/bench_fork${fk}_$rep.log 2>&1
    echo "exit $?" >> $O/bench_fork${fk}_$rep.log
  done
done
