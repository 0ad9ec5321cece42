#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
for v in 296 444 592 888; do
  echo "== vec blocks $v"
  export TF_VEC_BLOCKS=$v
  TF_PCG_RESIDENT=0 TF_PCG_FUSED=0 timeout 600 python scripts/cg_protocols.py "cantilever:5/3:fp32" "cantilever:5/3:fp64" "torsion:1:fp32" "torsion:1:fp64" "cantilever:17/6:fp32" 2>&1 | grep '"graph"' | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['problem'], d['iterations'], round(d['us_per_iteration'], 2))"
done
