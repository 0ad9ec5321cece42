#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
for i in 1 2; do python scripts/simp_c1_probe.py; done
TF_PCG_RES_BY=4 python scripts/simp_c1_probe.py
TF_PCG_RES_BY=8 python scripts/simp_c1_probe.py
TF_TILE_AUTOTUNE=0 python scripts/simp_c1_probe.py
