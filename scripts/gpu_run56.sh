#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_operator.py tests/test_gpu_solver.py -q -p no:cacheprovider --timeout 300 -rf -k "edof or general or atomic or colo" > gpurun_out/pytest_e57.txt 2>&1
tail -2 gpurun_out/pytest_e57.txt
for v1 in 0; do for dn in 0 1; do for c in c2 c4 c5 c5f64; do
  r=$(TF_EDOF_DENSE=$dn TF_EDOF_V1=$v1 timeout 300 python bench.py --config $c --kernel edof --scatter parallel_atomic --steps 50 --warmup 5 --no-simp --no-cpu 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['ms_per_step']*1e3,1), round(d['roofline']['frac'],3))")
  echo "dense=$dn $c: GDOF/s us frac = $r"
done; done; done
timeout 600 ncu --set full --clock-control none -k regex:k_edof_staged -s 5 -c 1 -o gpurun_out/prof_edof4_c5 python bench.py --config c5 --kernel edof --scatter parallel_atomic --steps 10 --warmup 3 --no-simp --no-cpu > gpurun_out/ncu_edof2.log 2>&1
