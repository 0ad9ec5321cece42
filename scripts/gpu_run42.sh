#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
mkdir -p gpurun_out
timeout 1200 python scripts/simp_presets.py torsion:1 cantilever:5/3:10 cantilever:17/6:4 > gpurun_out/simp_presets42.txt 2>&1
timeout 600 python -m pytest tests/test_slab.py -m gpu -q -p no:cacheprovider --timeout 300 -rf > gpurun_out/pytest_slab42.txt 2>&1
for c in c2 c5; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_grid_tile5 -s 100 -c 1 -o gpurun_out/prof_tile5d_$c python bench.py --config $c --steps 10 --warmup 60 --no-simp --no-cpu > gpurun_out/ncu_tile5d_$c.log 2>&1
done
cat gpurun_out/simp_presets42.txt; tail -2 gpurun_out/pytest_slab42.txt
