#!/bin/bash
# round-2 final validation: all GPU tests, smoke, bench lines (default, persistent), reference arm,
# ncu --set full of the dominant kernel (B1, MN-major weights)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/final2
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/final2/gpu_tests.log 2>&1
echo "gpu tests exit $?" >> gpurun_out/final2/gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final2/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/final2/smoke.log
timeout 900 python bench.py > gpurun_out/final2/bench_default.log 2>&1
echo "exit $?" >> gpurun_out/final2/bench_default.log
timeout 900 python bench.py --recurrence 1 --no-cpu-baseline > gpurun_out/final2/bench_persistent.log 2>&1
echo "exit $?" >> gpurun_out/final2/bench_persistent.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final2/bench_reference.log 2>&1
echo "exit $?" >> gpurun_out/final2/bench_reference.log
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:EpiB1IO -s 300 -c 1 \
  -o /tmp/prof_b1 python tools/one_step.py 2 > gpurun_out/final2/ncu_b1.log 2>&1
ncu -i /tmp/prof_b1.ncu-rep --page raw --csv > gpurun_out/final2/b1_raw.csv 2>/dev/null
python tools/ncu_hot.py /tmp/prof_b1.ncu-rep 25 > gpurun_out/final2/b1_hot.txt 2>&1
ls gpurun_out/final2
