#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python tools/gemm_one.py 2 4096 4096 8192 256 > gpurun_out/g2.log 2>&1 && python tools/gemm_one.py 1 4096 4096 8192 256 >> gpurun_out/g2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_tc2 -s 1 -c 1 -o gpurun_out/prof_tc2 python tools/gemm_one.py 2 4096 4096 8192 256 > gpurun_out/ncu_tc2.log 2>&1 ; \
ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 1 -c 1 -o gpurun_out/prof_tc1 python tools/gemm_one.py 1 4096 4096 8192 256 > gpurun_out/ncu_tc1.log 2>&1
cat gpurun_out/g2.log; tail -3 gpurun_out/ncu_tc2.log
