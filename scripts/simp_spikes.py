"""Per-iteration walls of the device SIMP loop at c4 (phase 1 of
default_schedule(120)), repeated, with and without Python GC."""
import gc
import os
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
for mode in ("gc", "nogc", "gc"):
    if mode == "nogc":
        gc.disable()
    else:
        gc.enable()
    r = run_simp(pb, SimpConfig(schedule=sched(8), precision=prec))
    torch.cuda.synchronize()
    print(mode, [round(h.wall_s * 1e3, 1) for h in r.history], [h.cg_iterations for h in r.history])
