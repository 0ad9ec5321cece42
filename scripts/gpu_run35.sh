#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
mkdir -p gpurun_out
timeout 300 python scripts/simp_c2_probe.py 4 > gpurun_out/simp35.txt 2>&1
TF_PCG_TRACE=1 timeout 300 python scripts/simp_c2_probe.py 2 >> gpurun_out/simp35.txt 2>&1
TF_PCG_RESIDENT=0 timeout 300 python scripts/simp_c2_probe.py 4 >> gpurun_out/simp35.txt 2>&1
cat gpurun_out/simp35.txt | cut -c1-400
