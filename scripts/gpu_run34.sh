#!/bin/bash
# round-1 evidence refresh: full gpu suite, default bench (with SIMP c1/c2 + CG), ncu of tile5 and the resident PCG
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -rf > gpurun_out/pytest_gpu34.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke34.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench34_default.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench34.csv python bench.py --steps 20 --warmup 3 --no-simp --no-cpu > gpurun_out/ncu_launch34.log 2>&1
for c in c2 c5; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_grid_tile5 -s 5 -c 1 -o gpurun_out/prof_tile5_$c python bench.py --config $c --steps 10 --warmup 3 --no-simp --no-cpu > gpurun_out/ncu_tile5_$c.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pcg_resident -c 1 -o gpurun_out/prof_resident_c2 python scripts/cg_protocols.py cantilever:1:fp32 > gpurun_out/ncu_res_c2.log 2>&1
tail -3 gpurun_out/pytest_gpu34.txt; tail -1 gpurun_out/smoke34.txt; tail -1 gpurun_out/bench34_default.txt | head -c 600; ls gpurun_out/*.ncu-rep
