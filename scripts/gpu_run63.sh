#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
timeout 900 python -m pytest tests/test_gpu_operator.py tests/test_gpu_solver.py -q -p no:cacheprovider --timeout 300 -rf 2>&1 | grep -v "^E  " | tail -40
