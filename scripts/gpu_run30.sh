#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
mkdir -p gpurun_out
TF_PCG_TRACE=1 timeout 300 python scripts/cg_protocols.py c1:1:fp64 cantilever:0.2:fp64 cantilever:1:fp32 cantilever:1:fp64 torsion:1:fp32 > gpurun_out/cgproto30.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_resident.py -q -p no:cacheprovider --timeout 300 -rf -x > gpurun_out/pytest_res30.txt 2>&1
tail -2 gpurun_out/pytest_res30.txt; grep "resident\|tf_pcg" gpurun_out/cgproto30.txt | awk 'NR%5==1 || /protocol/'
