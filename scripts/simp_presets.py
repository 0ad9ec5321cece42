"""SIMP wall-clock on the paper's presets (Tables 4-5 protocol:
default_schedule(120), FP32 fused operator), optionally truncated to the first
N iterations for the largest meshes.  Prints one JSON line per run.

usage: python scripts/simp_presets.py preset:scale[:n_iter[:prec]] ...
"""
from __future__ import annotations

import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_18020_b200 import SimpConfig, default_schedule, make_preset, run_simp  # noqa: E402
from paper_2604_18020_b200.simp import ContinuationSchedule  # noqa: E402
from paper_2604_18020_b200.solver import pcg_protocol  # noqa: E402

for spec in sys.argv[1:]:
    parts = spec.split(":")
    name, scale = parts[0], float(eval(parts[1]))
    n = int(parts[2]) if len(parts) > 2 else 120
    prec = parts[3] if len(parts) > 3 else "fp32"
    pb = make_preset(name, scale)
    full = default_schedule(120)
    if n < 120:
        ph = full.phases[0]
        sched = ContinuationSchedule((type(ph)(1, n, p=ph.p, beta=ph.beta, move=ph.move, rmin_end=ph.rmin_end),),
                                     full.rmin_start)
    else:
        sched = full
    ph = full.phases[0]
    warm = ContinuationSchedule((type(ph)(1, 1, p=ph.p, beta=ph.beta, move=ph.move, rmin_end=ph.rmin_end),), 1.5)
    run_simp(pb, SimpConfig(schedule=warm, precision=prec))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = run_simp(pb, SimpConfig(schedule=sched, precision=prec))
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    its = [h.cg_iterations for h in res.history]
    print(json.dumps({"preset": name, "scale": scale, "n_elem": pb.mesh.n_elem, "precision": prec,
                      "simp_iterations": n, "wall_s": wall, "s_per_iter": wall / n,
                      "median_iter_s": float(np.median([h.wall_s for h in res.history])),
                      "total_cg": int(sum(its)), "capped_solves": int(sum(i >= 1000 for i in its)),
                      "final_compliance": res.history[-1].compliance,
                      "selected_compliance": res.selected.compliance if res.selected else None}), flush=True)
