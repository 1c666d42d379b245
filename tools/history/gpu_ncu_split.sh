#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
{ for e in 1 2 3 4; do python tools/gemm_one.py $e 256 4096 4096 256; done; python tools/gemm_one.py 1 256 4096 4096 64; } > gpurun_out/split.log 2>&1
python tools/gemm_one.py 3 256 4096 4096 0 >> gpurun_out/split.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_tc2s -s 1 -c 1 -o gpurun_out/prof_tc2s python tools/gemm_one.py 3 256 4096 4096 0 > gpurun_out/ncu_tc2s.log 2>&1
cat gpurun_out/split.log
