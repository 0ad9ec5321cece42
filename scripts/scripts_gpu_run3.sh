#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
for c in c2 c5; do
timeout 300 python bench.py --config $c --kernel tile --steps 100 --warmup 5 --no-simp --no-cpu > gpurun_out/bench_${c}_tile.json 2>&1
done
timeout 600 python bench.py --steps 200 --warmup 10 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_grid_tile -s 5 -c 1 -o gpurun_out/prof_tile_c5 python bench.py --config c5 --steps 10 --warmup 3 --no-simp --no-cpu > gpurun_out/ncu_tile_c5.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_simp.csv python -c "
import numpy as np
from paper_2604_18020_b200 import *
pb = make_preset('cantilever', 0.4)
op = MatFreeOperator(pb.mesh, build_edof(pb.mesh), pb.bcs, np.full(pb.mesh.n_elem, 0.5), SimpParams(3.0), 'fp32')
u, rep = solve_equilibrium(op, pb.bcs.force, CgConfig(max_iter=30))
print(rep.iterations)
" > gpurun_out/ncu_cg.log 2>&1
ls -la gpurun_out
