#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
mkdir -p gpurun_out
c=c5f64
oz=$(timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-simp --no-cpu 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['config']['launch']['z_chunk']); import sys; print(d['ms_per_step']*1e3, d['config']['launch'], file=sys.stderr)")
echo "$c production oz=$oz"
TF_TILE_AUTOTUNE=0 TF_TILE_OZ=$oz timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_grid_tile5 -s 8 -c 1 -o gpurun_out/tile5_prod_$c -f python bench.py --config $c --steps 10 --warmup 3 --no-simp --no-cpu > gpurun_out/ncu_$c.log 2>&1
tail -1 gpurun_out/ncu_$c.log | cut -c1-200
