#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
mkdir -p gpurun_out
timeout 1200 python scripts/bf16_negative.py 0.2 1/3 2/3 1.0 > gpurun_out/bf16neg45.txt 2>&1
cat gpurun_out/bf16neg45.txt | cut -c1-900
