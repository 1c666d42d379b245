#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for rot in 1 0; do
  echo "== MLSTM_RC_ROTATE=$rot" >> gpurun_out/r2g_trace.log
  MLSTM_RC_ROTATE=$rot timeout 300 python tools/trace_recur.py 2>&1 | grep -v "^ *[0-9]" >> gpurun_out/r2g_trace.log
done
# application-replay ncu of the forward kernel with a few metrics (kernel replay breaks the persistent kernel)
timeout 900 ncu --replay-mode application --clock-control none -k regex:fwd_recur -s 1 -c 1 \
  --metrics gpu__time_duration.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,dram__bytes_read.sum,l1tex__m_xbar2l1tex_read_bytes.sum \
  python tools/one_step.py 2 > gpurun_out/r2g_ncu.log 2>&1
echo "ncu exit $?" >> gpurun_out/r2g_ncu.log
