#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; tail gpurun_out/plain.log; exit 1; }
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:EpiB2 -s 300 -c 1 -o gpurun_out/prof3_B2 $CMD > gpurun_out/ncu3.log 2>&1
echo done
