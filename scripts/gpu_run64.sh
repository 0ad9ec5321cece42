#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -rf 2>&1 | tail -3
for gen in 0 1; do TF_TILE_GENERIC=$gen TF_PCG_TRACE=1 timeout 300 python scripts/cg_protocols.py c1:1:fp64 cantilever:1:fp32 cantilever:1:fp64 2>&1 | grep "resident\|tf_pcg" | awk 'NR%4==1 || /protocol/' | cut -c1-200; done
python scripts/simp_c1_probe.py
