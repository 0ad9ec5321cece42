#!/bin/bash
# SM-resident PCG: parity tests + protocol timings
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_resident.py -q -p no:cacheprovider --timeout 300 -rf -x > gpurun_out/pytest_res23.txt 2>&1
timeout 600 python scripts/cg_protocols.py c1:1:fp64 cantilever:0.2:fp64 cantilever:1:fp32 cantilever:1:fp64 torsion:1:fp32 torsion:1:fp64 > gpurun_out/cgproto23.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -rf > gpurun_out/pytest_gpu23.txt 2>&1
tail -3 gpurun_out/pytest_res23.txt; cat gpurun_out/cgproto23.txt; tail -3 gpurun_out/pytest_gpu23.txt
