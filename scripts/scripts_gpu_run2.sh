#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
for k in tile pull; do for c in c2 c5; do
timeout 300 python bench.py --config $c --kernel $k --steps 100 --warmup 5 --no-simp --no-cpu > gpurun_out/bench_${c}_${k}.json 2>&1
done; done
timeout 600 python bench.py --steps 200 --warmup 10 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_grid_tile -s 5 -c 1 -o gpurun_out/prof_tile_c5 python bench.py --config c5 --steps 10 --warmup 3 --no-simp --no-cpu > gpurun_out/ncu_tile_c5.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_grid_tile -s 5 -c 1 -o gpurun_out/prof_tile_c2 python bench.py --config c2 --steps 10 --warmup 3 --no-simp --no-cpu > gpurun_out/ncu_tile_c2.log 2>&1
ls -la gpurun_out
