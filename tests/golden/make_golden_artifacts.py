"""Report-artifact goldens (history CSV, SIMP summary JSON, selected density
snapshot) written by the REAL reference's cmd_simp (cli.py:250-297) for a
fixed synthetic SimpResult (run_simp patched out so wall times are fixed).
Run in the build container only:

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_artifacts.py
"""

from __future__ import annotations

import shutil
import sys
import tempfile
from pathlib import Path

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent / "artifacts"


def synthetic_result(mod_simp, problem, config):
    """Same values as tests/test_host.py::_synthetic_result (any package's dataclasses)."""
    rng = np.random.default_rng(5)
    hist = []
    for it in range(1, 7):
        hist.append(mod_simp.IterationRecord(
            it, float(50.0 / it + rng.uniform()), float(rng.uniform()), int(100 + 7 * it), bool(it % 3),
            1.5 if it < 3 else 3.0, float(2 ** (it // 2)), 0.2, 1.5 - 0.01 * it, 0.3 + 1e-7 * it,
            it == 5, 0.125 * it + 1e-10))
    n = problem.mesh.n_elem
    sel = mod_simp.SelectedRecord(4, 12.345678912345, 0.2, rng.uniform(size=n), rng.uniform(size=n),
                                  rng.uniform(size=problem.mesh.n_dof), 3.0, 2.0)
    return mod_simp.SimpResult(hist, sel, 1, rng.uniform(size=n), rng.uniform(size=n), 742, 3.25, config,
                               problem.name)


def main():
    sys.path.insert(0, REF_SRC)
    import topofuse.cli as cli
    from topofuse import simp

    cli.run_simp = lambda problem, config: synthetic_result(simp, problem, config)
    tmp = Path(tempfile.mkdtemp())
    cfg = dict(cli.DEFAULTS) if hasattr(cli, "DEFAULTS") else {}
    cfg.update(preset="cantilever", scale=0.1, iters=6, precision="fp64", variant="fused", scatter="serial",
               seed=42, cg_cap=1000, backend=None, out=str(tmp))
    cli.cmd_simp(cfg)
    OUT.mkdir(exist_ok=True)
    for f in sorted(tmp.iterdir()):
        shutil.copy(f, OUT / f.name)
        print(f.name, f.stat().st_size)


if __name__ == "__main__":
    main()
