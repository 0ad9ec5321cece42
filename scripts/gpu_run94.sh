#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
time (timeout 600 python -m pytest tests/test_slab.py -q -p no:cacheprovider --timeout 500 -m gpu -k peer 2>&1 | grep -E "^E |passed|failed|Error|Timeout" | head -20)
