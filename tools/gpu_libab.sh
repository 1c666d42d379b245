#!/bin/bash
# interleaved A/B of two builds of libmlstm.so (ab/libmlstm_A.so vs ab/libmlstm_B.so), C3 bench
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
CFG=${1:-C3}; R=${2:-3}
{
for r in $(seq 1 $R); do
for x in A B; do
  MLSTM_LIB=ab/libmlstm_$x.so timeout 600 python bench.py --config $CFG --steps 30 --warmup 5 --no-cpu-baseline --no-e2e | python3 -c "
import sys,json; d=json.loads(sys.stdin.read()); p=d['phases_ms_per_step']; c=d['clocks']
print('$x', round(d['value']), 'ms', round(d['ms_per_step'],2), 'fwd', p['fwd_rec'], 'bwd', p['bwd_rec'], 'wgrad', p['wgrad'], 'opt', p['optimizer'], 'ce', p['ce'], 'mhz', c['sm_mhz'], 'per_mhz', round(d['value']/c['sm_mhz']) if c['sm_mhz'] else None)"
done; done
} > gpurun_out/libab.log 2>&1
cat gpurun_out/libab.log
