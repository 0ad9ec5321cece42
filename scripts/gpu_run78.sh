#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
timeout 900 python -m pytest tests/test_slab.py tests/test_slab_simp.py tests/test_gpu_operator.py tests/test_gpu_solver.py -q -p no:cacheprovider --timeout 600 -m gpu 2>&1 | grep -E "^E |passed|failed|Error" | head -30
