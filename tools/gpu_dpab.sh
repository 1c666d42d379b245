#!/bin/bash
# N-GPU interleaved A/B of two builds (ab/libmlstm_A.so vs B) on C3 and C5
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
N=${1:-2}
{
timeout 900 python -m pytest tests/test_gpu_dp.py -q -x 2>&1 | tail -2
for cfg in C3 C5; do for x in A B A B; do
  MLSTM_LIB=ab/libmlstm_$x.so timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29551 bench.py --config $cfg --gpus $N --steps 6 --warmup 3 --no-e2e 2>&1 | grep "^{" | python3 -c "
import sys,json; d=json.loads(sys.stdin.read()); p=d['phases_ms_per_step']; print('$cfg $x', round(d['value']), 'ms', round(d['ms_per_step'],2), 'wgrad', p['wgrad'], 'allreduce', p['allreduce'], d['clocks']['sm_mhz'])"
done; done
} > gpurun_out/dpab.log 2>&1
cat gpurun_out/dpab.log
