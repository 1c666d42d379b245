#!/bin/bash
# dW_dec before BPTT (+ its allreduce bucket first): full GPU suite incl. DP on 2 GPUs, N=2 bench
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r2ad_tests.log 2>&1
echo "gpu tests exit $?" >> gpurun_out/r2ad_tests.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 \
  bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r2ad_bench2.log 2>&1
echo "exit $?" >> gpurun_out/r2ad_bench2.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2ad_bench1.log 2>&1
echo "exit $?" >> gpurun_out/r2ad_bench1.log
