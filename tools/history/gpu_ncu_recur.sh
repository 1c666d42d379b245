#!/bin/bash
# ncu --set full of the two persistent recurrence kernels (one capture each) + the summary metrics
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out/ncur
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/ncur/plain.log 2>&1 || exit 1
for K in fwd_recur_kernel bwd_recur_kernel; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$K -s 1 -c 1 -o /tmp/pr_$K $CMD > gpurun_out/ncur/$K.log 2>&1
  ncu -i /tmp/pr_$K.ncu-rep --page raw --csv > gpurun_out/ncur/${K}_raw.csv 2>/dev/null
  python tools/ncu_hot.py /tmp/pr_$K.ncu-rep 25 > gpurun_out/ncur/${K}_hot.txt 2>&1
  cp /tmp/pr_$K.ncu-rep gpurun_out/ncur/ 2>/dev/null
done
ls -la gpurun_out/ncur
