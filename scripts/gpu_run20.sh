#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_solver.py -q -p no:cacheprovider --timeout 600 -rf -k "general_connectivity" > gpurun_out/pytest_general.txt 2>&1
python scripts/pcie_probe.py > gpurun_out/pcie.txt 2>&1
for tool in memcheck racecheck synccheck; do
timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_smoke.py > gpurun_out/sanitizer_$tool.txt 2>&1; echo "rc=$?" >> gpurun_out/sanitizer_$tool.txt
done
ls gpurun_out | head
