"""Generate the golden fixtures in tests/golden/ by running the REAL reference.

Run in the build container only (the reference does not exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache NUMBA_NUM_THREADS=1 \
        python tests/golden/make_golden.py [--simp]

It imports the unmodified reference package from /root/reference/pkg/src
(read-only) and records, for seeded inputs:

  ke.npz          unit_stiffness(0.3) (element.py:69-101), bitwise
  matvec_*.npz    MatFreeOperator.apply outputs (operator.py:90-117) with the
                  numba backend, fused/three_stage x fp64/fp32, serial scatter;
                  plus diagonal() and element_energies()
  hashes.json     sha256 of reference outputs at sizes too large to store
                  (c1 48x24x24 and c2 120x60x30), so bitwise parity of the
                  oracle can be pinned at full size from a few bytes
  cg.json         cold-solve anchors (solve_equilibrium, solver.py:150-183):
                  iterations, termination, compliance, residual histories
  simp_*.npz      run_simp trajectories (simp.py:324-448): per-iteration
                  compliance / CG counts and final densities (--simp only)

Inputs are regenerated in the tests from the same seeds with numpy's
default_rng, so only outputs are stored.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent


def _sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def matvec_case(tf, dims, seed, p=3.0):
    m = tf.StructuredMesh(*dims)
    edof = tf.build_edof(m)
    bcs = tf.cantilever_bcs(m)
    rng = np.random.default_rng(seed)
    rho = rng.uniform(0.05, 1.0, m.n_elem)
    v = rng.standard_normal(m.n_dof)
    rec = {"edof_sha": _sha(edof), "fixed": np.asarray(bcs.fixed_dofs)}
    for prec in ("fp64", "fp32"):
        for variant in ("fused", "three_stage"):
            op = tf.MatFreeOperator(m, edof, bcs, rho, tf.SimpParams(p), prec, variant,
                                    "serial", backend="numba")
            rec[f"apply_{variant}_{prec}"] = op.apply(v.astype(op.precision.dtype))
        op = tf.MatFreeOperator(m, edof, bcs, rho, tf.SimpParams(p), prec, "fused", "serial",
                                backend="numba")
        rec[f"diag_{prec}"] = op.diagonal()
        # raw kernel contract: fused_serial on an unmasked input, accumulate
        out = np.zeros(m.n_dof, dtype=op.precision.dtype)
        op.kernels.fused_serial(edof, op.ke, op.scale, v.astype(op.precision.dtype), out)
        rec[f"raw_fused_{prec}"] = out
    op = tf.MatFreeOperator(m, edof, bcs, rho, tf.SimpParams(p), "fp64", backend="numba")
    rec["energies"] = op.element_energies(v)
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--simp", action="store_true", help="also record SIMP trajectories (slow)")
    args = ap.parse_args()
    sys.path.insert(0, REF_SRC)
    import topofuse as tf
    import numba

    assert numba.get_num_threads() == 1, "run with NUMBA_NUM_THREADS=1 for serial goldens"

    np.savez(OUT / "ke.npz", ke=tf.unit_stiffness(0.3))

    # small meshes: full outputs stored
    for dims, seed in [((4, 3, 2), 11), ((5, 3, 2), 12), ((1, 1, 1), 1001), ((24, 12, 6), 42)]:
        rec = matvec_case(tf, dims, seed)
        tag = "x".join(map(str, dims))
        np.savez_compressed(OUT / f"matvec_{tag}.npz", seed=seed, dims=np.array(dims),
                            **{k: v for k, v in rec.items() if k != "edof_sha"})
        meta = json.loads((OUT / "hashes.json").read_text()) if (OUT / "hashes.json").exists() else {}
        meta[f"edof_{tag}"] = rec["edof_sha"]
        (OUT / "hashes.json").write_text(json.dumps(meta, indent=1, sort_keys=True))
        print("matvec", tag, flush=True)

    # larger meshes: hashes + norms only
    meta = json.loads((OUT / "hashes.json").read_text())
    for dims, seed in [((48, 24, 24), 42), ((120, 60, 30), 42)]:
        rec = matvec_case(tf, dims, seed)
        tag = "x".join(map(str, dims))
        meta[f"edof_{tag}"] = rec["edof_sha"]
        for k, v in rec.items():
            if k in ("edof_sha", "fixed"):
                continue
            meta[f"{k}_{tag}"] = {"sha256": _sha(v), "norm": float(np.linalg.norm(v.astype(np.float64))),
                                  "sum": float(np.sum(v.astype(np.float64)))}
        print("hash", tag, flush=True)
    (OUT / "hashes.json").write_text(json.dumps(meta, indent=1, sort_keys=True))

    # cold CG anchors, rho = 0.5, p = 3 (PAPER Table 8 protocol)
    cg = {}
    for name, scale in [("desk", 0.2), ("s30", 1 / 30), ("s15", 1 / 15), ("80x40x20", 2 / 3),
                        ("c2", 1.0)]:
        pb = tf.make_preset("cantilever", scale)
        edof = tf.build_edof(pb.mesh)
        for prec in ("fp64", "fp32"):
            if name == "c2" and prec == "fp32":
                continue
            op = tf.MatFreeOperator(pb.mesh, edof, pb.bcs, np.full(pb.mesh.n_elem, 0.5),
                                    tf.SimpParams(3.0), prec, "fused", "serial", backend="numba")
            t0 = time.perf_counter()
            u, rep = tf.solve_equilibrium(op, pb.bcs.force, tf.CgConfig())
            cg[f"{name}_{prec}"] = {
                "dims": [pb.mesh.nelx, pb.mesh.nely, pb.mesh.nelz],
                "iterations": rep.iterations, "termination": rep.termination,
                "converged": rep.converged, "rel_residual": rep.rel_residual,
                "verified": rep.verified_rel_residual, "compliance": rep.compliance,
                "matvecs": rep.matvecs,
                "history": [float(h) for h in rep.residual_history],
                "wall_s": time.perf_counter() - t0,
            }
            print("cg", name, prec, rep.iterations, rep.termination, rep.compliance, flush=True)
    # torsion c3 fp64 anchor
    pb = tf.make_preset("torsion", 1.0)
    op = tf.MatFreeOperator(pb.mesh, tf.build_edof(pb.mesh), pb.bcs, np.full(pb.mesh.n_elem, 0.5),
                            tf.SimpParams(3.0), "fp64", "fused", "serial", backend="numba")
    u, rep = tf.solve_equilibrium(op, pb.bcs.force, tf.CgConfig())
    cg["torsion_fp64"] = {"dims": [pb.mesh.nelx, pb.mesh.nely, pb.mesh.nelz],
                          "iterations": rep.iterations, "termination": rep.termination,
                          "compliance": rep.compliance, "rel_residual": rep.rel_residual,
                          "history": [float(h) for h in rep.residual_history]}
    print("cg torsion", rep.iterations, rep.compliance, flush=True)
    (OUT / "cg.json").write_text(json.dumps(cg, indent=1))

    if args.simp:
        simp_goldens(tf)


def simp_goldens(tf):
    from topofuse.simp import ContinuationSchedule, Phase

    def record(res, path, extra):
        h = res.history
        np.savez_compressed(
            path,
            compliance=np.array([r.compliance for r in h]),
            cg_iterations=np.array([r.cg_iterations for r in h]),
            cg_converged=np.array([r.cg_converged for r in h]),
            grayness=np.array([r.grayness for r in h]),
            volume=np.array([r.volume for r in h]),
            restarted=np.array([r.restarted for r in h]),
            rho_phys=res.rho_phys, rho_raw=res.rho_raw,
            selected_compliance=np.nan if res.selected is None else res.selected.compliance,
            selected_iteration=-1 if res.selected is None else res.selected.iteration,
            total_cg=res.total_cg_iterations, wall_s=res.wall_s, **extra,
        )

    # config c1: 48x24x24 cantilever, single phase p=3, beta=1, move 0.2, rmin 1.5, 30 its
    m = tf.StructuredMesh(48, 24, 24)
    pb = tf.ProblemPreset("cantilever", m, tf.cantilever_bcs(m), 0.3, 1.5)
    sched = ContinuationSchedule(phases=(Phase(1, 30, p=3.0, beta=1.0, move=0.2, rmin_end=1.5),),
                                 rmin_start=1.5)
    for prec in ("fp64",):
        res = tf.run_simp(pb, tf.SimpConfig(schedule=sched, precision=prec, scatter="serial"))
        record(res, OUT / f"simp_c1_{prec}.npz", {})
        print("simp c1", prec, res.wall_s, res.total_cg_iterations, res.history[-1].compliance,
              flush=True)
    # desk 24x12x6, default_schedule(120), fused serial (conftest.py:18-37)
    desk = tf.make_preset("cantilever", 0.2)
    for prec in ("fp64", "fp32"):
        res = tf.run_simp(desk, tf.SimpConfig(schedule=tf.default_schedule(120), precision=prec,
                                              variant="fused", scatter="serial"))
        record(res, OUT / f"simp_desk_{prec}.npz", {})
        print("simp desk", prec, res.wall_s, res.selected.compliance, flush=True)


if __name__ == "__main__":
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    main()
