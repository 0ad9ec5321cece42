#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
for c in c2 c3 c4 c5 c2f64 c5f64; do
timeout 300 python bench.py --config $c --steps 100 --warmup 5 --no-simp --no-cpu > gpurun_out/bench_${c}.json 2>&1
done
timeout 900 python bench.py --steps 200 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_grid_tile -s 5 -c 1 -o gpurun_out/prof_tile3_c5 python bench.py --config c5 --steps 10 --warmup 3 --no-simp --no-cpu > gpurun_out/ncu_tile3_c5.log 2>&1
ls gpurun_out | head -50
