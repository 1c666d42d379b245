#!/bin/bash
# ncu evidence for the C3 step: launch list (1 step) and --set full captures of the top kernels;
# the reports are summarised on the box (raw metrics + hottest source lines) to stay under the
# 64 MiB copy-back limit
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out/ncu
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/ncu/plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -s 1060 -c 1100 --csv --log-file gpurun_out/ncu/launches.csv $CMD > gpurun_out/ncu/list.log 2>&1
for K in ${KERNELS:-EpiF2IO EpiB1 EpiF1 EpiB2 EpiWgrad}; do
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:$K -s ${SKIP:-20} -c 1 -o /tmp/prof_$K $CMD > gpurun_out/ncu/$K.log 2>&1
  ncu -i /tmp/prof_$K.ncu-rep --page raw --csv > gpurun_out/ncu/${K}_raw.csv 2>/dev/null
  python tools/ncu_hot.py /tmp/prof_$K.ncu-rep 40 > gpurun_out/ncu/${K}_hot.txt 2>&1
  ncu -i /tmp/prof_$K.ncu-rep --page source --csv > /tmp/src_$K.csv 2>/dev/null && gzip -c /tmp/src_$K.csv > gpurun_out/ncu/${K}_source.csv.gz
done
du -sh gpurun_out/ncu; ls gpurun_out/ncu
