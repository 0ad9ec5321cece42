"""SIMP golden for a degenerate 4-step default schedule, from the REAL
reference.  Run in the build container only:

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache NUMBA_NUM_THREADS=1 \
        python tests/golden/make_golden_short_schedule.py

default_schedule(4) jumps p 1.5 -> 3.5 -> 4.5 and beta 1 -> 32 in four steps
on the desk cantilever (24x12x6): the compliance reaches ~2e8 and |u| ~ 2e8,
where element energies evaluated as u^T Ke u carry rounding of size
eps*|Ke|*|u|^2 (the reference's own minimum energy is -5.4).  The golden pins
that the B200 loop runs through this regime like the reference (no spurious
'positive sensitivity' rejection) with the same compliance history.
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
    res = tf.run_simp(pb, tf.SimpConfig(schedule=tf.simp.default_schedule(4)))
    out = dict(compliance=[r.compliance for r in res.history],
               cg_iterations=[r.cg_iterations for r in res.history],
               volume=[r.volume for r in res.history],
               restarted=[r.restarted for r in res.history])
    (OUT / "simp_short_schedule.json").write_text(json.dumps(out, indent=1) + "\n")
    print(out)


if __name__ == "__main__":
    main()
