#!/bin/bash
# round 2: 2-GPU data-parallel tests + bench N=2 (both recurrence implementations)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/r2dp2_smi.txt
timeout 1200 python -m pytest tests/test_gpu_dp.py "tests/test_gpu_parity.py::test_loss_scale_invariance" -q > gpurun_out/r2dp2_tests.log 2>&1
echo "dp tests exit $?" >> gpurun_out/r2dp2_tests.log
for rc in 0 1; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 2 --steps 20 --warmup 5 --recurrence $rc >> gpurun_out/r2dp2_bench.log 2>&1
  echo "N=2 recurrence=$rc exit $?" >> gpurun_out/r2dp2_bench.log
done
