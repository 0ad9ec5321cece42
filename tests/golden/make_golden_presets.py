"""SIMP goldens on the other benchmark presets (torsion, mbb, bridge), from the
REAL reference.  Run in the build container only:

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache NUMBA_NUM_THREADS=1 \
        python tests/golden/make_golden_presets.py

Protocol (as config c1, BASELINE.json): single continuation phase p=3, beta=1,
move 0.2, rmin 1.5, 30 iterations, fused serial scatter, presets at the desk
scale 0.2 (torsion 33x11x11, mbb 30x10x5, bridge 30x10x5).  Records the
per-iteration compliance / CG counts and the final densities.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent


def main():
    sys.path.insert(0, REF_SRC)
    import numba

    import topofuse as tf
    from topofuse.simp import ContinuationSchedule, Phase

    assert numba.get_num_threads() == 1
    sched = ContinuationSchedule(phases=(Phase(1, 30, p=3.0, beta=1.0, move=0.2, rmin_end=1.5),), rmin_start=1.5)
    for name, precs in (("torsion", ("fp64", "fp32")), ("mbb", ("fp64",)), ("bridge", ("fp64",))):
        pb = tf.make_preset(name, 0.2)
        for prec in precs:
            res = tf.run_simp(pb, tf.SimpConfig(schedule=sched, precision=prec, scatter="serial"))
            h = res.history
            np.savez_compressed(
                OUT / f"simp_{name}_{prec}.npz",
                compliance=np.array([r.compliance for r in h]),
                cg_iterations=np.array([r.cg_iterations for r in h]),
                volume=np.array([r.volume for r in h]),
                rho_phys=res.rho_phys, total_cg=res.total_cg_iterations)
            print(name, prec, res.wall_s, res.total_cg_iterations, h[-1].compliance, flush=True)


if __name__ == "__main__":
    main()
