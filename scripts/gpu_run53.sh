#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
TF_BENCH_SAME_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 3 --no-simp --no-cpu > gpurun_out/bench53_2rank.txt 2>&1
echo "rc=$?"; tail -3 gpurun_out/bench53_2rank.txt | cut -c1-700
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 1 --steps 20 --warmup 3 --no-simp --no-cpu > gpurun_out/bench53_1rank.txt 2>&1
echo "rc=$?"; tail -1 gpurun_out/bench53_1rank.txt | cut -c1-300
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29535 bench.py --impl reference --gpus 2 --steps 2 --warmup 3 > gpurun_out/bench53_ref2.txt 2>&1
echo "rc=$?"; tail -2 gpurun_out/bench53_ref2.txt | cut -c1-300
