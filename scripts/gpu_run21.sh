#!/bin/bash
# x-range tile launches + slab split on GPU, full gpu suite, racecheck outside the graph
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -rf > gpurun_out/pytest_gpu21.txt 2>&1
TF_PCG_NOGRAPH=1 timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python scripts/sanitize_smoke.py > gpurun_out/sanitizer_racecheck_nograph.txt 2>&1; echo "rc=$?" >> gpurun_out/sanitizer_racecheck_nograph.txt
for c in c2 c5; do timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-simp --no-cpu > gpurun_out/bench21_$c.txt 2>&1; done
tail -3 gpurun_out/pytest_gpu21.txt
