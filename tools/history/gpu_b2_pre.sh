cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x > gpurun_out/b2pre_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/b2pre_tests.log
sed -i 's/--steps 10 --warmup 3/--steps 30 --warmup 5/' tools/gpu_libab.sh
bash tools/gpu_libab.sh C3 4
