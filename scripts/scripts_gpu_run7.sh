#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
for c in c2 c5; do
timeout 300 python bench.py --config $c --steps 100 --warmup 5 --no-simp --no-cpu > gpurun_out/bench_${c}_tile.json 2>&1
done
timeout 900 python bench.py --steps 200 --warmup 10 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 20 --warmup 3 --no-simp --no-cpu > gpurun_out/ncu_launch.log 2>&1
for c in c2 c5; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_grid_tile -s 5 -c 1 -o gpurun_out/prof_tile3_$c python bench.py --config $c --steps 10 --warmup 3 --no-simp --no-cpu > gpurun_out/ncu_tile3_$c.log 2>&1
done
cat > gpurun_out/cg_prof.py <<'PY'
import sys, numpy as np
from paper_2604_18020_b200 import *
scale = float(sys.argv[1]); prec = sys.argv[2]
pb = make_preset('cantilever', scale)
op = MatFreeOperator(pb.mesh, build_edof(pb.mesh), pb.bcs, np.full(pb.mesh.n_elem, 0.5), SimpParams(3.0), prec)
u, rep = solve_equilibrium(op, pb.bcs.force, CgConfig(max_iter=12))
print(rep.iterations)
PY
for sc in 1.0 2.8333333333333335; do
TF_PCG_NOGRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_cg_$sc.csv python gpurun_out/cg_prof.py $sc fp32 > gpurun_out/ncu_cg_$sc.log 2>&1
done
ls -la gpurun_out
