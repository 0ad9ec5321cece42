#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
timeout 900 python -m pytest tests/test_gpu_operator.py tests/test_slab.py -q -p no:cacheprovider --timeout 600 -m gpu -x 2>&1 | grep -E "^E |passed|failed|Error" | head -20
for sz in 0 1; do for c in c2 c3 c4 c5; do
  r=$(TF_TILE_SPLITZ=$sz timeout 300 python bench.py --config $c --steps 200 --warmup 5 --no-simp --no-cpu 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['ms_per_step']*1e3,2), round(d.get('warm_l2_ms_per_step',0)*1e3,2), d['config'].get('launch'))")
  echo "splitz=$sz $c: GDOF/s us(flushed) us(warm) = $r"
done; done
