#!/bin/bash
# final round-1 validation on 2 GPUs: all GPU tests, smoke, bench lines (C3 default with cpu baseline
# and e2e, C3 N=2, C4, C5, weight norm)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
{
echo "== tests"; timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
echo "== C3 default"; timeout 900 python bench.py
echo "== C3 N=2"; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 2>&1 | grep "^{"
echo "== C4"; timeout 1200 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline
echo "== C5"; timeout 900 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline
echo "== C3 weight norm"; timeout 900 python bench.py --weight-norm --no-cpu-baseline --steps 10 --warmup 3
} > gpurun_out/final.log 2>&1
grep -v "^{" gpurun_out/final.log
grep "^{" gpurun_out/final.log | python3 -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['config']['workload'][:60], d['n_gpus'], round(d['value']), 'e2e', round(d['e2e']['value']) if d.get('e2e') else None, 'frac', round(d['roofline']['frac'],3), d['clocks'])"
