#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
timeout 600 python scripts/cg_protocols.py "cantilever:5/3:fp32" "cantilever:1:fp32" "cantilever:17/6:fp32" 2>&1 | tail -12
timeout 300 python bench.py --config c4 --steps 200 --warmup 5 --no-simp --no-cpu 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c4 matvec us', d['ms_per_step']*1e3, d['value'])"
