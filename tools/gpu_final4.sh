#!/bin/bash
# round-2 closing validation after the F2 register preload: all GPU tests, smoke, default bench (5 + 50 steps),
# ncu launch list (-> kernel shares) + --set full of the dominant kernel (B1), reference arm
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/final4; mkdir -p $O
timeout 1200 python -m pytest tests -q -m gpu > $O/gpu_tests.log 2>&1
echo "gpu tests exit $?" >> $O/gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke exit $?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_default.log 2>&1
echo "exit $?" >> $O/bench_default.log
CMD="python tools/one_step.py 2"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 1100 -c 1100 --csv \
  --log-file $O/launches.csv $CMD > $O/list.log 2>&1
python tools/launch_summary.py $O/launches.csv > $O/launch_summary.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:EpiB1IO -s 300 -c 1 -o /tmp/prof_b1 $CMD > $O/b1.log 2>&1
ncu -i /tmp/prof_b1.ncu-rep --page raw --csv > $O/EpiB1IO_raw.csv 2>/dev/null
python tools/ncu_hot.py /tmp/prof_b1.ncu-rep 30 > $O/EpiB1IO_hot.txt 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.log 2>&1
echo "exit $?" >> $O/bench_reference.log
du -sh $O
