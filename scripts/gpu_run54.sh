#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_resident.py -q -p no:cacheprovider --timeout 300 -rf -x > gpurun_out/pytest_res54.txt 2>&1
tail -2 gpurun_out/pytest_res54.txt
for by in 0 8 16; do TF_PCG_RES_BY=$by TF_PCG_TRACE=1 timeout 300 python scripts/cg_protocols.py c1:1:fp64 cantilever:1:fp32 torsion:1:fp32 2>&1 | grep "tf_pcg_res\|resident" | awk 'NR%4==1 || /protocol/' | cut -c1-260; done
for by in 4 8; do TF_PCG_RES_BY=$by TF_PCG_TRACE=1 timeout 300 python scripts/cg_protocols.py c1:1:fp64 cantilever:1:fp64 2>&1 | grep "tf_pcg_res\|resident" | awk 'NR%4==1 || /protocol/' | cut -c1-260; done
