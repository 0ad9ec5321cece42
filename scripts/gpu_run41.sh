#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -rf > gpurun_out/pytest_gpu41.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke41.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench41_default.txt 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench41_ref.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench41.csv python bench.py --steps 20 --warmup 3 --no-simp --no-cpu > gpurun_out/ncu_launch41.log 2>&1
for c in c2 c5; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_grid_tile5 -s 40 -c 1 -o gpurun_out/prof_tile5c_$c python bench.py --config $c --steps 10 --warmup 3 --no-simp --no-cpu > gpurun_out/ncu_tile5c_$c.log 2>&1
done
tail -3 gpurun_out/pytest_gpu41.txt; tail -1 gpurun_out/smoke41.txt; tail -1 gpurun_out/bench41_default.txt | head -c 300; echo; tail -1 gpurun_out/bench41_ref.txt | head -c 300
