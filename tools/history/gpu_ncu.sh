#!/bin/bash
# ncu evidence for the C3 step: launch list (1 step) and --set full captures of the top kernels
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; tail gpurun_out/plain.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -s 1060 -c 1100 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1
for K in EpiF2 EpiB1 EpiF1 EpiB2; do
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:$K -s 20 -c 1 -o gpurun_out/prof_$K $CMD > gpurun_out/ncu_$K.log 2>&1
done
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:EpiWgrad -s 0 -c 2 -o gpurun_out/prof_wgrad $CMD > gpurun_out/ncu_wgrad.log 2>&1
ls -la gpurun_out
