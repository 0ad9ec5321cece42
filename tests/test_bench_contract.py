"""The bench.py JSON line keeps the driver's contract: checked on the last
committed B200 line (profiles/bench_r2_c2.json, written by `python bench.py`)."""

from __future__ import annotations

import json

import numpy as np
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_bench_line_has_the_contract_keys():
    d = json.loads((ROOT / "profiles" / "bench_r2_c2.json").read_text())
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
              "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["warmup"] >= 3 and d["higher_is_better"] is True
    assert "workload" in d["config"] and "l2" in d["config"]
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor") and r["unit"] in ("GB/s", "TFLOP/s")
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert "traffic" in r
    c = d["cpu_baseline"]
    assert c["kind"] in ("port", "reference") and c["cores"] >= 1 and c["value"] > 0 and c["sample"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] >= d["steps"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    bad = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    assert not bad & set(d["clocks"]["reasons"])


def test_bench_cli_defaults():
    """No flags -> N = 1 and a K/W that finish within minutes (driver contract)."""
    import re

    src = (ROOT / "bench.py").read_text()
    assert re.search(r'add_argument\("--gpus", type=int, default=1\)', src)
    assert re.search(r'add_argument\("--steps", type=int, default=\d+\)', src)
    assert re.search(r'add_argument\("--warmup", type=int, default=(\d+)\)', src)
    assert int(re.search(r'add_argument\("--warmup", type=int, default=(\d+)\)', src).group(1)) >= 3


def test_slab_problem_matches_global_cantilever():
    """bench.slab_problem (the c5w weak-scaling slab, built without global
    arrays) gives each rank the constraints and load of the global cantilever
    restricted to its slab, and both replicas of an interface plane the same
    input values."""
    import bench
    from paper_2604_18020_b200.mesh import StructuredMesh, cantilever_bcs
    from paper_2604_18020_b200.slab import SlabPartition

    gdims = (9, 4, 3)
    gm = StructuredMesh(*gdims)
    gb = cantilever_bcs(gm)
    parts = []
    for world in (1, 2, 3):
        parts = [bench.slab_problem(gdims, world, r) for r in range(world)]
        for r, (_, part, lb, rho, v) in enumerate(parts):
            want = SlabPartition(gm, world, r).local_bcs(gb)
            assert np.array_equal(lb.fixed_dofs, want.fixed_dofs)
            assert np.array_equal(lb.force, want.force)
            assert rho.shape == (part.local_mesh.n_elem,) and v.shape == (part.local_mesh.n_dof,)
        for r in range(world - 1):
            pl, pr = parts[r][1], parts[r + 1][1]
            assert np.array_equal(parts[r][4][pl.plane_dofs(pl.local_mesh.nelx)],
                                  parts[r + 1][4][pr.plane_dofs(0)])
