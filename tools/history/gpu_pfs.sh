#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
{
timeout 120 python tools/diag_step.py mixed 1024 64 256 16 || echo "DIAG FAILED rc=$?"
for pf in 0 1; do
  echo "== PF_STASH=$pf"; MLSTM_PF_STASH=$pf timeout 600 python tools/trace_step.py 2>&1 | grep -v Warn | grep -v nanmean | head -5
  MLSTM_PF_STASH=$pf timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['phases_ms_per_step']['fwd_rec'], d['phases_ms_per_step']['bwd_rec'], d['clocks'])"
done
} > gpurun_out/pfs.log 2>&1
cat gpurun_out/pfs.log
