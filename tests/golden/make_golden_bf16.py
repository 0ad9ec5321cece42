"""Golden fixtures for the emulated-BF16 path, produced by the REAL reference.

Run in the build container only (the reference does not exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache NUMBA_NUM_THREADS=1 \
        python tests/golden/make_golden_bf16.py

Imports the unmodified reference (/root/reference/pkg/src, read-only) and
records for seeded inputs (same seeds as make_golden.py's matvec cases):

  bf16_<dims>.npz   round_to_bf16 of special values (precision.py:65-85);
                    MatFreeOperator(precision="bf16").apply (fused/three_stage,
                    serial scatter), diagonal(), apply_fp64();
                    raw fused_serial_bf16 / gemm_bf16 / jacobi_diag_bf16
  bf16_solve.json   desk cantilever cold solves in bf16 (solve_equilibrium,
                    solver.py:150-183: recompute disabled for quantized
                    operators) and iterative refinement (solve_refined,
                    solver.py:211-262) -- the paper's negative result anchors
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent

SPECIALS = np.array([0.0, -0.0, 1.0, 1.00390625, 1.005859375, 1.0029296875, 3.0e38, 3.4e38, -7.5e-39,
                     1e-40, np.inf, -np.inf, np.nan, 65504.0, -1.2345678, 0.1], dtype=np.float32)


def main():
    sys.path.insert(0, REF_SRC)
    import numba

    import topofuse as tf
    from topofuse import precision as P

    assert numba.get_num_threads() == 1, "run with NUMBA_NUM_THREADS=1 for serial goldens"
    for dims, seed in (((4, 3, 2), 11), ((5, 3, 2), 1030)):
        m = tf.StructuredMesh(*dims)
        edof = tf.build_edof(m)
        bcs = tf.cantilever_bcs(m)
        rng = np.random.default_rng(seed)
        rho = rng.uniform(0.05, 1.0, m.n_elem)
        v = rng.standard_normal(m.n_dof)
        rec = {"specials": SPECIALS, "round_specials": P.round_to_bf16(SPECIALS)}
        for variant in ("fused", "three_stage"):
            op = tf.MatFreeOperator(m, edof, bcs, rho, tf.SimpParams(3.0), "bf16", variant, "serial",
                                    backend="numba")
            rec[f"apply_{variant}"] = op.apply(v.astype(np.float32))
        op = tf.MatFreeOperator(m, edof, bcs, rho, tf.SimpParams(3.0), "bf16", "fused", "serial",
                                backend="numba")
        rec["diag"] = op.diagonal()
        rec["apply_fp64"] = op.apply_fp64(v)
        vq = P.round_to_bf16(v.astype(np.float32))
        out = np.zeros(m.n_dof, dtype=np.float32)
        op.kernels.fused_serial_bf16(edof, op.ke, op.scale, vq, out)
        rec["raw_fused_serial_bf16"] = out
        rec["raw_gemm_bf16"] = op.kernels.gemm_bf16(op.kernels.gather(edof, vq), op.ke, op.scale)
        d = np.zeros(m.n_dof, dtype=np.float32)
        op.kernels.jacobi_diag_bf16(edof, np.diag(op.ke).copy(), op.scale, d)
        rec["raw_jacobi_bf16"] = d
        np.savez_compressed(OUT / f"bf16_{dims[0]}x{dims[1]}x{dims[2]}.npz", **rec)

    pb = tf.make_preset("cantilever", 0.2)
    rho = np.full(pb.mesh.n_elem, 0.5)
    edof = tf.build_edof(pb.mesh)
    solves = {}
    for prec in ("bf16", "fp32"):
        op = tf.MatFreeOperator(pb.mesh, edof, pb.bcs, rho, tf.SimpParams(3.0), prec, backend="numba")
        u, rep = tf.solve_equilibrium(op, pb.bcs.force, tf.CgConfig())
        solves[f"desk_{prec}"] = {"iterations": rep.iterations, "termination": rep.termination,
                                  "compliance": rep.compliance,
                                  "verified_rel_residual": rep.verified_rel_residual,
                                  "history": [float(h) for h in rep.residual_history]}
    op32 = tf.MatFreeOperator(pb.mesh, edof, pb.bcs, rho, tf.SimpParams(3.0), "fp32", backend="numba")
    op16 = tf.MatFreeOperator(pb.mesh, edof, pb.bcs, rho, tf.SimpParams(3.0), "bf16", backend="numba")
    u, ir = tf.solve_refined(op32, op16, pb.bcs.force)
    solves["desk_ir"] = {"converged": ir.converged, "stagnated": ir.stagnated, "outer_steps": ir.outer_steps,
                         "inner_iterations": ir.inner_iterations, "outer_residuals": ir.outer_residuals,
                         "compliance": ir.compliance}
    (OUT / "bf16_solve.json").write_text(json.dumps(solves, indent=1))
    print("wrote bf16 fixtures")


if __name__ == "__main__":
    main()
