#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
mkdir -p gpurun_out
for t4 in 0 1; do for c in c2 c3 c4 c5; do
  r=$(TF_TILE4=$t4 timeout 300 python bench.py --config $c --steps 200 --warmup 5 --no-simp --no-cpu 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['ms_per_step']*1e3,2), round(d.get('warm_l2_ms_per_step',0)*1e3,2))")
  echo "tile4=$t4 $c: GDOF/s us(flushed) us(warm) = $r"
done; done
