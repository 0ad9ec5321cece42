#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
mkdir -p gpurun_out
for oz in 0 2 4 5 6 8 11; do for c in c2 c3; do
  r=$(TF_TILE_OZ=$oz timeout 300 python bench.py --config $c --steps 200 --warmup 5 --no-simp --no-cpu 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['ms_per_step']*1e3,2), round(d.get('warm_l2_ms_per_step',0)*1e3,2))")
  echo "oz=$oz $c: GDOF/s us(flushed) us(warm) = $r"
done; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_grid_tile5 -s 5 -c 1 -o gpurun_out/prof_tile5b_c2 python bench.py --config c2 --steps 10 --warmup 3 --no-simp --no-cpu > gpurun_out/ncu_tile5b_c2.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_edof_fused -s 5 -c 1 -o gpurun_out/prof_edof_c5 python bench.py --config c5 --kernel edof --scatter parallel_atomic --steps 10 --warmup 3 --no-simp --no-cpu > gpurun_out/ncu_edof_c5.log 2>&1
ls gpurun_out/*.ncu-rep
