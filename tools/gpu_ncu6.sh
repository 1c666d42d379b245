#!/bin/bash
# round-2 ncu evidence: launch list of C3 steps (default per-timestep path) + --set full of the
# dominant kernel (B1), F2 and the weight-gradient GEMM; summaries written on the box
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out/ncu6
CMD="python tools/one_step.py 2"
$CMD > gpurun_out/ncu6/plain.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 1100 -c 1100 --csv \
  --log-file gpurun_out/ncu6/launches.csv $CMD > gpurun_out/ncu6/list.log 2>&1
python tools/launch_summary.py gpurun_out/ncu6/launches.csv > gpurun_out/ncu6/launch_summary.txt 2>&1
for K in EpiB1IO EpiF2IO; do
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:$K -s 300 -c 1 -o /tmp/prof_$K $CMD > gpurun_out/ncu6/$K.log 2>&1
  ncu -i /tmp/prof_$K.ncu-rep --page raw --csv > gpurun_out/ncu6/${K}_raw.csv 2>/dev/null
  python tools/ncu_hot.py /tmp/prof_$K.ncu-rep 30 > gpurun_out/ncu6/${K}_hot.txt 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:EpiWgrad -s 3 -c 1 -o /tmp/prof_wg $CMD > gpurun_out/ncu6/wgrad.log 2>&1
ncu -i /tmp/prof_wg.ncu-rep --page raw --csv > gpurun_out/ncu6/wgrad_raw.csv 2>/dev/null
python tools/ncu_hot.py /tmp/prof_wg.ncu-rep 30 > gpurun_out/ncu6/wgrad_hot.txt 2>&1
du -sh gpurun_out/ncu6; ls gpurun_out/ncu6
