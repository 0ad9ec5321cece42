#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
for lib in libtopofuse_b200.so libtopofuse_b200_minb4.so; do for c in c2 c5; do
TOPOFUSE_B200_LIB=$GRAFT_REPO_ROOT/paper_2604_18020_b200/lib/$lib timeout 300 python bench.py --config $c --steps 100 --warmup 5 --no-simp --no-cpu > gpurun_out/bench_${c}_$lib.json 2>&1
done; done
TF_BENCH_SAME_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 3 --no-simp --no-cpu > gpurun_out/bench_2rank_samedev.json 2>&1
timeout 900 python bench.py --steps 200 --warmup 10 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_grid_tile -s 5 -c 1 -o gpurun_out/prof_tile3_c5 python bench.py --config c5 --steps 10 --warmup 3 --no-simp --no-cpu > gpurun_out/ncu_tile3_c5.log 2>&1
ls -la gpurun_out
