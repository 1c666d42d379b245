#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
{
echo "== default"; timeout 900 python bench.py
echo "== weight norm"; timeout 900 python bench.py --weight-norm --no-cpu-baseline --steps 10 --warmup 3 | python3 -c "
import sys,json; d=json.loads(sys.stdin.read()); print('WN', round(d['value']), d['phases_ms_per_step'], d['clocks'])"
echo "== reference"; timeout 900 python bench.py --impl reference --steps 2 --warmup 3
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')"
} > gpurun_out/run16.log 2>&1
cat gpurun_out/run16.log
