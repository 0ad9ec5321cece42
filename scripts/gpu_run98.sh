#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
for lib in lib lib_minb4; do for c in c2 c3 c4 c5; do
  r=$(TOPOFUSE_B200_LIB=$GRAFT_REPO_ROOT/paper_2604_18020_b200/$lib/libtopofuse_b200.so timeout 300 python bench.py --config $c --steps 200 --warmup 5 --no-simp --no-cpu 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['ms_per_step']*1e3,2), d['config'].get('launch'))")
  echo "$lib $c: $r"
done; done
