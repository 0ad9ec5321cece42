"""SIMP golden for the projected-volume OC variant (SimpConfig.volume_on =
"projected", simp.py:393-401 of the reference), from the REAL reference.
Run in the build container only:

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache NUMBA_NUM_THREADS=1 \
        python tests/golden/make_golden_projected.py

Desk cantilever (24x12x6), default_schedule(12) (beta reaches 32), FP64.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

REF_SRC = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent


def main():
    sys.path.insert(0, REF_SRC)
    import topofuse as tf

    pb = tf.make_preset("cantilever", 0.2)
    res = tf.run_simp(pb, tf.SimpConfig(schedule=tf.simp.default_schedule(12), volume_on="projected"))
    out = dict(compliance=[r.compliance for r in res.history],
               cg_iterations=[r.cg_iterations for r in res.history],
               volume=[r.volume for r in res.history],
               restarted=[r.restarted for r in res.history],
               rho_phys_mean=float(res.rho_phys.mean()))
    (OUT / "simp_projected.json").write_text(json.dumps(out, indent=1) + "\n")
    print(out)


if __name__ == "__main__":
    main()
