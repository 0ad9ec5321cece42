#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
python scripts/pcie_probe.py none
python scripts/pcie_probe.py tf
timeout 900 python -m pytest tests/test_gpu_operator.py -q -p no:cacheprovider --timeout 300 -rf -k "stream" 2>&1 | tail -2
for c in c2 c5; do
  r=$(timeout 300 python bench.py --config $c --steps 200 --warmup 5 --no-simp --no-cpu 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value'],2), d['e2e'])")
  echo "$c: $r"
done
