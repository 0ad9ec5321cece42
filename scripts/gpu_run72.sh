#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
timeout 600 python -m pytest tests/test_gpu_operator.py tests/test_gpu_solver.py -q -p no:cacheprovider --timeout 300 -rf -k "general or contract or three_stage or edof" 2>&1 | tail -3
for col in 0 1; do for c in c2 c5 c5f64; do
  r=$(TF_EDOF_COLORED=$col timeout 300 python bench.py --config $c --kernel edof --scatter serial --steps 30 --warmup 3 --no-simp --no-cpu 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['ms_per_step']*1e3,1))")
  echo "colored=$col $c serial: GDOF/s us = $r"
done; done
