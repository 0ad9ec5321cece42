#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
nvidia-smi -q -d PCIE 2>&1 | grep -i "gen\|width\|link" | head -12
./scripts/h2d_probe
for i in 1 2 3; do
  r=$(timeout 300 python bench.py --config c2 --steps 200 --warmup 5 --no-simp --no-cpu 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value'],2), d['e2e']['value'])")
  echo "c2 run $i: $r"
done
nvidia-smi -q -d PCIE 2>&1 | grep -i "gen\|width" | head -6
