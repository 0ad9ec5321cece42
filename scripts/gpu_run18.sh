#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf -x > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 900 python bench.py --steps 200 > gpurun_out/bench.json 2> gpurun_out/bench.err
TF_PCG_UNFUSED=1 timeout 900 python bench.py --steps 50 --no-cpu > gpurun_out/bench_unfused.json 2> gpurun_out/bench_unfused.err
timeout 900 python - > gpurun_out/simp_c2.txt 2>&1 <<'PY'
import time, numpy as np, torch
from paper_2604_18020_b200 import *
from paper_2604_18020_b200.simp import ContinuationSchedule, Phase
for scale, n in ((1.0, 10), (17/6, 3)):
    pb = make_preset('cantilever', scale)
    sched = default_schedule(120)
    ph = sched.phases[0]
    short = ContinuationSchedule((Phase(1, n, ph.p, ph.beta, ph.move, ph.rmin_end),), sched.rmin_start)
    t0 = time.perf_counter()
    res = run_simp(pb, SimpConfig(schedule=short, precision='fp32'))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(scale, pb.mesh.n_elem, 's/iter', dt / n, [round(h.wall_s, 4) for h in res.history], [h.cg_iterations for h in res.history])
PY
for sc in 1.0 2.8333333333333335; do
TF_PCG_NOGRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_cg_$sc.csv python scripts/cg_prof.py $sc fp32 > gpurun_out/ncu_cg_$sc.log 2>&1
done
ls gpurun_out | head -50
