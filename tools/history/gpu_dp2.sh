#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
{
nvidia-smi -L
timeout 600 python -m pytest tests/test_gpu_dp.py -q -x 2>&1 | tail -15
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 10 --warmup 3
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()"
} > gpurun_out/dp2.log 2>&1
tail -30 gpurun_out/dp2.log
