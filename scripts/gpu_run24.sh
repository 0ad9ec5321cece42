#!/bin/bash
# resident PCG v2 (sentinel-slot exchange, lean layout, trace)
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_resident.py -q -p no:cacheprovider --timeout 300 -rf -x > gpurun_out/pytest_res24.txt 2>&1
TF_PCG_TRACE=1 timeout 600 python scripts/cg_protocols.py c1:1:fp64 cantilever:0.2:fp64 cantilever:1:fp32 cantilever:1:fp64 torsion:1:fp32 torsion:1:fp64 > gpurun_out/cgproto24.txt 2>&1
for oz in 3 4 6 8; do TF_PCG_RES_OZ=$oz TF_PCG_TRACE=1 timeout 300 python scripts/cg_protocols.py cantilever:1:fp32 >> gpurun_out/cgproto24_oz.txt 2>&1; done
TF_PCG_RES_LEAN=1 TF_PCG_TRACE=1 timeout 300 python scripts/cg_protocols.py c1:1:fp64 cantilever:1:fp32 >> gpurun_out/cgproto24_oz.txt 2>&1
tail -3 gpurun_out/pytest_res24.txt; grep -v skipped gpurun_out/cgproto24.txt | grep -v '"graph"\|fused_graph'; grep "tf_pcg_res\|resident" gpurun_out/cgproto24_oz.txt
