"""Per-iteration desk SIMP trace (device glue, host glue, exact kernel) vs the golden."""
import numpy as np
from paper_2604_18020_b200 import SimpConfig, default_schedule, make_preset, run_simp
g = np.load("tests/golden/simp_desk_fp64.npz")
pb = make_preset("cantilever", 0.2)
cfg = SimpConfig(schedule=default_schedule(120), precision="fp64")
runs = {"device": run_simp(pb, cfg, device_glue=True), "host": run_simp(pb, cfg, device_glue=False)}
import os
os.environ["TOPOFUSE_B200_EXACT"] = "1"
runs["host_exact"] = run_simp(pb, cfg, device_glue=False)
for k, r in runs.items():
    c = np.array([h.compliance for h in r.history])
    its = np.array([h.cg_iterations for h in r.history])
    rel = np.abs(c - g["compliance"]) / g["compliance"]
    first = int(np.argmax(rel > 1e-6)) if np.any(rel > 1e-6) else -1
    print(k, "selected", r.selected.compliance, r.selected.iteration, "golden", float(g["selected_compliance"]),
          int(g["selected_iteration"]), "first>1e-6 at", first, "max rel", rel.max())
    print("  rel by 10s:", [f"{x:.1e}" for x in rel[::10]])
    print("  cg its diff:", (its - g["cg_iterations"])[:40].tolist())
