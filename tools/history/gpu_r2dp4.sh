#!/bin/bash
# round 2: 4-GPU data-parallel tests + bench lines (C3 both recurrences, C5 at the paper LR)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_dp.py -q > gpurun_out/r2dp4_tests.log 2>&1
echo "dp tests exit $?" >> gpurun_out/r2dp4_tests.log
for args in "--recurrence 0" "--recurrence 1" "--config C5"; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 \
    bench.py --gpus 4 --steps 20 --warmup 5 $args >> gpurun_out/r2dp4_bench.log 2>&1
  echo "N=4 $args exit $?" >> gpurun_out/r2dp4_bench.log
done
