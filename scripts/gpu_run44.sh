#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bf16.py -q -p no:cacheprovider --timeout 300 -rf > gpurun_out/pytest_bf16.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -rf > gpurun_out/pytest_gpu44.txt 2>&1
tail -30 gpurun_out/pytest_bf16.txt; tail -3 gpurun_out/pytest_gpu44.txt
