"""Device-time breakdown of device-resident SIMP iterations (torch.profiler /
CUPTI): which kernels, and how much of the loop's wall is not GPU work.
usage: python scripts/simp_iter_profile.py [cantilever scale] [prec]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2604_18020_b200 import SimpConfig, make_preset, run_simp  # noqa: E402
from paper_2604_18020_b200.simp import ContinuationSchedule, Phase  # noqa: E402

scale = float(eval(sys.argv[1])) if len(sys.argv) > 1 else 1.0
prec = sys.argv[2] if len(sys.argv) > 2 else "fp32"
pb = make_preset("cantilever", scale)
sched = lambda k: ContinuationSchedule((Phase(1, k, p=1.5, beta=1.0, move=0.2, rmin_end=1.5),), 1.5)  # noqa: E731
run_simp(pb, SimpConfig(schedule=sched(2), precision=prec))
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    t0 = time.perf_counter()
    res = run_simp(pb, SimpConfig(schedule=sched(3), precision=prec))
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
loop = sum(h.wall_s for h in res.history)
tot = {}
for e in prof.events():
    if e.device_type.name == "CUDA":
        k = e.name[:70]
        n, t = tot.get(k, (0, 0.0))
        tot[k] = (n + 1, t + e.device_time)
dev = sum(t for n, t in tot.values()) / 1e3
print(f"wall {wall*1e3:.1f} ms, loop {loop*1e3:.1f} ms (3 iterations), device {dev:.1f} ms; CG its {[h.cg_iterations for h in res.history]}")
for k, (n, t) in sorted(tot.items(), key=lambda kv: -kv[1][1])[:14]:
    print(f"{t/1e3/3:9.3f} ms/iter  {n:6d}x  {k}")
