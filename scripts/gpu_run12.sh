#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
for t3 in 0 1; do for c in c2 c4 c5; do
TF_TILE3=$t3 timeout 300 python bench.py --config $c --steps 100 --warmup 5 --no-simp --no-cpu > gpurun_out/bench_${c}_t3$t3.json 2>&1
done; done
timeout 300 python bench.py --config c5 --kernel edof --scatter parallel_atomic --steps 50 --warmup 5 --no-simp --no-cpu > gpurun_out/bench_c5_edof_atomic.json 2>&1
timeout 300 python bench.py --config c5 --kernel edof --scatter serial --steps 50 --warmup 5 --no-simp --no-cpu > gpurun_out/bench_c5_edof_colored.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_grid_tile -s 5 -c 1 -o gpurun_out/prof_tile4_c5 python bench.py --config c5 --steps 10 --warmup 3 --no-simp --no-cpu > gpurun_out/ncu_tile4_c5.log 2>&1
for sc in 1.0 2.8333333333333335; do
TF_PCG_NOGRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_cg_$sc.csv python scripts/cg_prof.py $sc fp32 > gpurun_out/ncu_cg_$sc.log 2>&1
done
ls -la gpurun_out
