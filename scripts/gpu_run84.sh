#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
timeout 600 python -m pytest tests/test_slab.py -q -p no:cacheprovider --timeout 300 -m gpu -k peer 2>&1 | grep -E "^E |passed|failed|Error|error" | head -30
