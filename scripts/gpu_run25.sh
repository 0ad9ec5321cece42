#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
mkdir -p gpurun_out
timeout 300 ./scripts/exchange_bench 2 256 2000 > gpurun_out/xchg25.txt 2>&1
for i in 1 2; do TF_PCG_TRACE=1 timeout 300 python scripts/cg_protocols.py c1:1:fp64 cantilever:1:fp32 cantilever:1:fp64 >> gpurun_out/cgproto25.txt 2>&1; done
cat gpurun_out/xchg25.txt; grep resident gpurun_out/cgproto25.txt
