#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_operator.py tests/test_gpu_solver.py -q -p no:cacheprovider --timeout 300 -rf -k "edof or general or three_stage or atomic or colo" > gpurun_out/pytest_e33.txt 2>&1
tail -2 gpurun_out/pytest_e33.txt
for dense in 0 1; do for c in c2 c5 c5f64; do for sc in parallel_atomic; do
  r=$(TF_EDOF_DENSE=$dense timeout 300 python bench.py --config $c --kernel edof --scatter $sc --steps 50 --warmup 5 --no-simp --no-cpu 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['ms_per_step']*1e3,1), round(d['roofline']['frac'],3))")
  echo "dense=$dense $c $sc: GDOF/s us frac = $r"
done; done; done
