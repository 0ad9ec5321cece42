#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 900 python bench.py --steps 200 --warmup 10 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python - > gpurun_out/simp_c2.txt 2>&1 <<'PY'
import time, numpy as np, torch
from paper_2604_18020_b200 import *
for scale, n in ((1.0, 10), (17/6, 3)):
    pb = make_preset('cantilever', scale)
    cfg = SimpConfig(schedule=default_schedule(120), precision='fp32')
    # first n iterations of the 120-iteration paper schedule
    sched = cfg.schedule
    from paper_2604_18020_b200.simp import ContinuationSchedule, Phase
    ph = sched.phases[0]
    short = ContinuationSchedule((Phase(1, n, ph.p, ph.beta, ph.move, ph.rmin_end),), sched.rmin_start)
    t0 = time.perf_counter()
    res = run_simp(pb, SimpConfig(schedule=short, precision='fp32'))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(scale, pb.mesh.n_elem, 's/iter', dt / n, [round(h.wall_s, 4) for h in res.history], [h.cg_iterations for h in res.history])
PY
ls -la gpurun_out
