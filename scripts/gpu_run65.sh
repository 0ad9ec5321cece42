#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
timeout 900 python -m pytest tests/test_gpu_solver.py -q -p no:cacheprovider --timeout 300 -rf -k "presets and torsion" 2>&1 | grep "^E  \|passed\|failed" | head -12 | cut -c1-400
TF_TILE_GENERIC=1 timeout 900 python -m pytest tests/test_gpu_solver.py -q -p no:cacheprovider --timeout 300 -rf -k "presets and torsion" 2>&1 | tail -1
