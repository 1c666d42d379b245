#!/bin/bash
# 4 GPUs: the NCCL data-parallel tests and the C3 N=4 bench line
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/dp4f; mkdir -p $O
timeout 1200 python -m pytest -q -m gpu tests/test_gpu_dp.py > $O/tests.log 2>&1
echo "tests exit $?" >> $O/tests.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 4 > $O/bench_n4.log 2>&1
echo "exit $?" >> $O/bench_n4.log
