#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
for pdl in 0 1 0 1; do
  echo "== PDL $pdl"
  TF_PCG_PDL=$pdl TF_PCG_RESIDENT=0 TF_PCG_FUSED=0 timeout 600 python scripts/cg_protocols.py "cantilever:5/3:fp32" "torsion:1:fp64" "cantilever:17/6:fp32" "cantilever:1:fp64" 2>&1 | grep '"graph"' | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['problem'], d['iterations'], round(d['us_per_iteration'], 2), d['compliance'])"
done
timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_resident.py -q -p no:cacheprovider --timeout 600 -m gpu 2>&1 | grep -E "^E |passed|failed" | head -4
