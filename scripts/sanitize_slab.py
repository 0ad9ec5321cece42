"""compute-sanitizer workload for the round's newer kernels in one process:
world-1 slab SIMP (slab CG step kernels, Jacobi partials, OC volumes/apply,
element halos), projected-volume device OC, parity-basis energies."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_18020_b200 import SimpConfig, default_schedule, make_preset, run_simp  # noqa: E402
from paper_2604_18020_b200.slab_simp import slab_run_simp  # noqa: E402

pb = make_preset("mbb", 0.2)
r = slab_run_simp(pb, SimpConfig(schedule=default_schedule(4)), device="cuda:0")
print("slab", [round(h.compliance, 4) for h in r.history])
r = run_simp(make_preset("cantilever", 0.2), SimpConfig(schedule=default_schedule(12), volume_on="projected"))
print("projected", [round(h.compliance, 4) for h in r.history])
