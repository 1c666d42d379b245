#!/bin/bash
# ncu --set full of the remaining SURVEY 8(d) kernels: input-projection table (a), decoder GEMM,
# CE (d), Adam (e), overflow scan
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out/ncu5
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/ncu5/plain.log 2>&1 || exit 1
for K in EpiTab EpiY ce_kernel adam_kernel overflow_kernel; do
  ncu --set full --clock-control none --kernel-name-base demangled -k regex:$K -s 1 -c 1 -o /tmp/p5_$K $CMD > gpurun_out/ncu5/$K.log 2>&1
  ncu -i /tmp/p5_$K.ncu-rep --page raw --csv > gpurun_out/ncu5/${K}_raw.csv 2>/dev/null
done
ls gpurun_out/ncu5
