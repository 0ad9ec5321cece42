"""Where a device-resident SIMP iteration spends its time (c4 by default):
cProfile of run_simp over a few phase-1 iterations after a warm-up run."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2604_18020_b200 import SimpConfig, make_preset, run_simp  # noqa: E402
from paper_2604_18020_b200.simp import ContinuationSchedule, Phase  # noqa: E402

scale = float(eval(sys.argv[1])) if len(sys.argv) > 1 else 5 / 3
prec = sys.argv[2] if len(sys.argv) > 2 else "fp32"
pb = make_preset("cantilever", scale)
sched = lambda k: ContinuationSchedule((Phase(1, k, p=1.5, beta=1.0, move=0.2, rmin_end=1.5),), 1.5)  # noqa: E731
run_simp(pb, SimpConfig(schedule=sched(2), precision=prec))
torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
res = run_simp(pb, SimpConfig(schedule=sched(4), precision=prec))
torch.cuda.synchronize()
pr.disable()
print("wall per iter", (time.perf_counter() - t0) / 4, [h.cg_iterations for h in res.history],
      [round(h.wall_s, 4) for h in res.history])
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
