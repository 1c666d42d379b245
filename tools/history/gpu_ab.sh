#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
{
timeout 120 python tools/diag_step.py mixed 1024 64 256 16 || echo "DIAG FAILED rc=$?"
echo "== tile"; timeout 600 python tools/trace_step.py 2>&1 | grep -v Warn | grep -v nanmean | head -6
echo "== row"; MLSTM_LIB=$PWD/paper_1808_01371_b200/libmlstm_row.so timeout 120 python tools/diag_step.py mixed 1024 64 256 16
MLSTM_LIB=$PWD/paper_1808_01371_b200/libmlstm_row.so timeout 600 python tools/trace_step.py 2>&1 | grep -v Warn | grep -v nanmean | head -6
} > gpurun_out/ab.log 2>&1
cat gpurun_out/ab.log
