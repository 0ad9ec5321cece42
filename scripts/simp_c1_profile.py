"""Where a c1 SIMP iteration goes (48x24x24, FP64, bench config): per-iteration
walls and CG counts, the CG share (CG iterations x the resident solve's
measured us/iteration) and a cProfile of the host side.
    python scripts/simp_c1_profile.py"""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2604_18020_b200 import (ContinuationSchedule, Phase, ProblemPreset, SimpConfig,  # noqa: E402
                                   StructuredMesh, cantilever_bcs, run_simp)

m = StructuredMesh(48, 24, 24)
pb = ProblemPreset("cantilever", m, cantilever_bcs(m), 0.3, 1.5)
sched = lambda k: ContinuationSchedule((Phase(1, k, p=3.0, beta=1.0, move=0.2, rmin_end=1.5),), 1.5)  # noqa: E731
run_simp(pb, SimpConfig(schedule=sched(2), precision="fp64"))
torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
res = run_simp(pb, SimpConfig(schedule=sched(30), precision="fp64"))
torch.cuda.synchronize()
pr.disable()
wall = time.perf_counter() - t0
cg = sum(h.cg_iterations for h in res.history)
print(f"wall per iter {1e3 * wall / 30:.3f} ms; CG iterations {cg} ({cg / 30:.0f} per SIMP iteration)")
print("walls", [round(1e3 * h.wall_s, 2) for h in res.history][:10])
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
