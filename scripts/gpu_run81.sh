#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
TF_PCG_NOGRAPH=1 timeout 300 python scripts/cg_kernel_times.py 5/3 fp32 2>&1 | grep -A6 protocol
TF_PCG_NOGRAPH=1 timeout 300 python scripts/cg_kernel_times.py 17/6 fp32 2>&1 | grep -A6 protocol
TF_PCG_NOGRAPH=1 timeout 300 python scripts/cg_kernel_times.py 1 fp32 2>&1 | grep -A6 protocol
