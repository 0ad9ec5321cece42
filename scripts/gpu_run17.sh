#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
for c in c2 c3 c4; do for oz in 0 2 3 4 5 6 8 10; do
TF_TILE_OZ=$oz timeout 300 python bench.py --config $c --steps 100 --warmup 5 --no-simp --no-cpu > gpurun_out/oz_${c}_$oz.json 2>&1
done; done
for oz in 0 12 16 24 32; do
TF_TILE_OZ=$oz timeout 300 python bench.py --config c5 --steps 100 --warmup 5 --no-simp --no-cpu > gpurun_out/oz_c5_$oz.json 2>&1
done
ls gpurun_out | head -80
