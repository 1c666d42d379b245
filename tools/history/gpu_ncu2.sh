#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; tail gpurun_out/plain.log; exit 1; }
for K in EpiF2 EpiB2 EpiF1; do
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:$K -s 300 -c 1 -o gpurun_out/prof2_$K $CMD > gpurun_out/ncu2_$K.log 2>&1
done
echo done
