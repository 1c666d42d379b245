#!/bin/bash
# final-state ncu evidence: launch list of one C3 step + --set full of the dominant kernels
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out/ncu4
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/ncu4/plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -s 1060 -c 1100 --csv --log-file gpurun_out/ncu4/launches.csv $CMD > gpurun_out/ncu4/list.log 2>&1
for K in EpiF2IO EpiB1IO EpiF1IO EpiB2; do
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:$K -s 20 -c 1 -o /tmp/prof_$K $CMD > gpurun_out/ncu4/$K.log 2>&1
  ncu -i /tmp/prof_$K.ncu-rep --page raw --csv > gpurun_out/ncu4/${K}_raw.csv 2>/dev/null
  python tools/ncu_hot.py /tmp/prof_$K.ncu-rep 30 > gpurun_out/ncu4/${K}_hot.txt 2>&1
done
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:EpiWgrad -s 0 -c 1 -o /tmp/prof_wg $CMD > gpurun_out/ncu4/wgrad.log 2>&1
ncu -i /tmp/prof_wg.ncu-rep --page raw --csv > gpurun_out/ncu4/wgrad_raw.csv 2>/dev/null
python tools/ncu_hot.py /tmp/prof_wg.ncu-rep 30 > gpurun_out/ncu4/wgrad_hot.txt 2>&1
du -sh gpurun_out/ncu4; ls gpurun_out/ncu4
