"""Per-iteration wall of the c2 SIMP (default_schedule phase 1, FP32): where the time goes."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2604_18020_b200 import SimpConfig, default_schedule, make_preset, run_simp
from paper_2604_18020_b200.simp import ContinuationSchedule

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4
prec = sys.argv[2] if len(sys.argv) > 2 else "fp32"
pb = make_preset("cantilever", 1.0)
ph = default_schedule(120).phases[0]
sched = ContinuationSchedule((type(ph)(1, n, p=ph.p, beta=ph.beta, move=ph.move, rmin_end=ph.rmin_end),), 1.5)
run_simp(pb, SimpConfig(schedule=ContinuationSchedule((type(ph)(1, 1, p=ph.p, beta=ph.beta, move=ph.move, rmin_end=ph.rmin_end),), 1.5), precision=prec))
torch.cuda.synchronize()
t0 = time.perf_counter()
res = run_simp(pb, SimpConfig(schedule=sched, precision=prec))
torch.cuda.synchronize()
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("TF_")}, "wall_s": time.perf_counter() - t0,
                  "iters": [(h.cg_iterations, round(h.wall_s * 1e3, 2)) for h in res.history]}))
