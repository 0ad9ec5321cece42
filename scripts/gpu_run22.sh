#!/bin/bash
# session-2 re-validation: full gpu suite, default bench, smoke, per-config kernel timings
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi22.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -rf > gpurun_out/pytest_gpu22.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke22.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench22_default.txt 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench22_ref.txt 2>&1
for c in c2 c5; do for k in tile edof; do timeout 300 python bench.py --config $c --kernel $k --steps 50 --warmup 5 --no-simp --no-cpu > gpurun_out/bench22_${c}_$k.txt 2>&1; done; done
tail -3 gpurun_out/pytest_gpu22.txt
