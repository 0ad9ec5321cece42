#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -rf > gpurun_out/pytest_gpu59.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke59.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench59_default.txt 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench59_ref.txt 2>&1
TF_PCG_TRACE=1 timeout 300 python scripts/cg_protocols.py c1:1:fp64 cantilever:1:fp32 > gpurun_out/cgproto59.txt 2>&1
tail -3 gpurun_out/pytest_gpu59.txt; tail -1 gpurun_out/smoke59.txt; tail -1 gpurun_out/bench59_ref.txt | cut -c1-200; grep "tf_pcg\|resident" gpurun_out/cgproto59.txt | awk 'NR%4==1 || /protocol/' | cut -c1-250
