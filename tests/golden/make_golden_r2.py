"""Round-2 golden fixtures: reference outputs at every BASELINE size the bench
times (run in the build container only; imports /root/reference/pkg/src
read-only).

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache NUMBA_NUM_THREADS=1 \
        python tests/golden/make_golden_r2.py {matvec,cg,simp} [names...]

  matvec  hashes_r2.json: sha256 / norm / sum / 4097 sampled entries of the
          reference apply (operator.py:90-117, numba fused_serial, FP32 and
          FP64) at c2 (120x60x30), c3 (torsion 165x55x55), c4 (200x100x50) and c5 (340x170x85)
          on the bench's seeded inputs (rho ~ U(0.05, 1), v ~ N(0, 1),
          default_rng(42); reference bench.py:161-173)
  cg      cg_r2.json: cold solve_equilibrium anchors (rho 0.5, p 3,
          CgConfig()) -- c2 FP32, c3 torsion FP32, c4 FP64/FP32
  simp    simp_c1_fp32.npz: config c1 (48x24x24, 30 its) in FP32, serial
          (name "atomic": simp_c1_fp32_atomic.npz, the same run with the
          reference's parallel_atomic scatter -- its own run-to-run spread)
"""

from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent
N_SAMPLE = 4097

MATVEC = {  # name: (preset, scale)
    "c2": ("cantilever", 1.0),
    "c3": ("torsion", 1.0),
    "c4": ("cantilever", 5 / 3),
    "c5": ("cantilever", 17 / 6),
}


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def sample_index(n):
    return np.unique(np.linspace(0, n - 1, N_SAMPLE).astype(np.int64))


def _merge(path, rec):
    d = json.loads(path.read_text()) if path.exists() else {}
    d.update(rec)
    path.write_text(json.dumps(d, indent=1, sort_keys=True))


def matvec(tf, names):
    out = {}
    for name in names:
        preset, scale = MATVEC[name]
        pb = tf.make_preset(preset, scale)
        m = pb.mesh
        edof = tf.build_edof(m)
        rng = np.random.default_rng(42)
        rho = rng.uniform(0.05, 1.0, m.n_elem)
        v = rng.standard_normal(m.n_dof)
        idx = sample_index(m.n_dof)
        for prec in ("fp32", "fp64"):
            op = tf.MatFreeOperator(m, edof, pb.bcs, rho, tf.SimpParams(3.0), prec, "fused", "serial",
                                    backend="numba")
            t0 = time.perf_counter()
            w = op.apply(v.astype(op.precision.dtype))
            out[f"apply_fused_{prec}_{name}"] = {
                "dims": [m.nelx, m.nely, m.nelz], "preset": preset, "scale": scale,
                "sha256": _sha(w), "norm": float(np.linalg.norm(w.astype(np.float64))),
                "sum": float(np.sum(w.astype(np.float64))), "max_abs": float(np.abs(w).max()),
                "sample": w[idx].astype(np.float64).tolist(), "s": time.perf_counter() - t0}
            print("matvec", name, prec, out[f"apply_fused_{prec}_{name}"]["s"], flush=True)
    _merge(OUT / "hashes_r2.json", out)


CG = {  # name: (preset, scale, precisions)
    "c2": ("cantilever", 1.0, ("fp32",)),
    "c3": ("torsion", 1.0, ("fp32",)),
    "c4": ("cantilever", 5 / 3, ("fp64", "fp32")),
}


def cg(tf, names):
    out = {}
    for name in names:
        preset, scale, precs = CG[name]
        pb = tf.make_preset(preset, scale)
        edof = tf.build_edof(pb.mesh)
        for prec in precs:
            op = tf.MatFreeOperator(pb.mesh, edof, pb.bcs, np.full(pb.mesh.n_elem, 0.5), tf.SimpParams(3.0),
                                    prec, "fused", "serial", backend="numba")
            t0 = time.perf_counter()
            u, rep = tf.solve_equilibrium(op, pb.bcs.force, tf.CgConfig())
            out[f"{name}_{prec}"] = {
                "dims": [pb.mesh.nelx, pb.mesh.nely, pb.mesh.nelz], "preset": preset, "scale": scale,
                "iterations": rep.iterations, "termination": rep.termination, "converged": rep.converged,
                "rel_residual": rep.rel_residual, "verified": rep.verified_rel_residual,
                "compliance": rep.compliance, "matvecs": rep.matvecs,
                "history": [float(h) for h in rep.residual_history], "wall_s": time.perf_counter() - t0}
            print("cg", name, prec, rep.iterations, rep.termination, rep.compliance,
                  out[f"{name}_{prec}"]["wall_s"], flush=True)
    _merge(OUT / "cg_r2.json", out)


def simp(tf, names):
    from topofuse.simp import ContinuationSchedule, Phase

    scatter, fname = ("parallel_atomic", "simp_c1_fp32_atomic.npz") if "atomic" in names else \
        ("serial", "simp_c1_fp32.npz")

    m = tf.StructuredMesh(48, 24, 24)
    pb = tf.ProblemPreset("cantilever", m, tf.cantilever_bcs(m), 0.3, 1.5)
    sched = ContinuationSchedule(phases=(Phase(1, 30, p=3.0, beta=1.0, move=0.2, rmin_end=1.5),),
                                 rmin_start=1.5)
    res = tf.run_simp(pb, tf.SimpConfig(schedule=sched, precision="fp32", scatter=scatter))
    h = res.history
    np.savez_compressed(
        OUT / fname,
        compliance=np.array([r.compliance for r in h]),
        cg_iterations=np.array([r.cg_iterations for r in h]),
        cg_converged=np.array([r.cg_converged for r in h]),
        volume=np.array([r.volume for r in h]),
        rho_phys=res.rho_phys, rho_raw=res.rho_raw,
        total_cg=res.total_cg_iterations, wall_s=res.wall_s)
    print("simp c1 fp32", scatter, res.wall_s, res.total_cg_iterations, h[-1].compliance, flush=True)


if __name__ == "__main__":
    sys.path.insert(0, REF_SRC)
    import topofuse as tf

    what = sys.argv[1]
    names = sys.argv[2:] or list({"matvec": MATVEC, "cg": CG, "simp": {"c1": 0}}[what])
    {"matvec": matvec, "cg": cg, "simp": simp}[what](tf, names)
