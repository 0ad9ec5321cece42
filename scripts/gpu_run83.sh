#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
timeout 1500 python -m pytest tests -q -p no:cacheprovider --timeout 900 -m gpu -x 2>&1 | grep -E "^E |passed|failed|Error" | head -20
timeout 600 python scripts/cg_protocols.py "c1:1:fp64" "cantilever:1:fp32" "cantilever:5/3:fp32" "torsion:1:fp64" "torsion:1:fp32" "cantilever:17/6:fp32" 2>&1 | grep -v skipped | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['problem'], d['protocol'], d['iterations'], round(d['us_per_iteration'], 2))"
