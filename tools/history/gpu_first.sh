#!/bin/bash
# first GPU contact: diagnostics then the GPU test-suite, every step under its own timeout
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
{
nvidia-smi -L
python -c "import torch;print(torch.cuda.get_device_name(0), torch.cuda.get_device_capability(0))"
timeout 300 python tools/diag_step.py fp32 64 64 4 16
MLSTM_DEBUG_SIMT_GEMM=1 timeout 300 python tools/diag_step.py mixed 64 64 4 16
timeout 120 python tools/diag_step.py mixed 64 64 4 16
timeout 120 python tools/diag_step.py mixed 128 64 130 5
timeout 300 python tools/diag_step.py mixed 1024 64 128 64
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -40
} > gpurun_out/first.log 2>&1
cat gpurun_out/first.log | tail -80
