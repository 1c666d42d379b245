#!/bin/bash
# round-2 final validation after the side-stream work: all GPU tests, smoke, default bench (5 + 50 steps), reference arm
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/final3; mkdir -p $O
timeout 2400 python -m pytest tests -q -m gpu > $O/gpu_tests.log 2>&1
echo "gpu tests exit $?" >> $O/gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke exit $?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_default.log 2>&1
echo "exit $?" >> $O/bench_default.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.log 2>&1
echo "exit $?" >> $O/bench_reference.log
