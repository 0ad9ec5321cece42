#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --steps 100 --no-cpu > gpurun_out/bench100.json 2> gpurun_out/bench100.err
for sc in 1.0 2.8333333333333335; do
TF_PCG_NOGRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_cg_$sc.csv python scripts/cg_prof.py $sc fp32 > gpurun_out/ncu_cg_$sc.log 2>&1
done
ls -la gpurun_out
