"""The documented BF16 negative result on B200 (north star; PAPER.md:1522-1552,
paper Table 6): emulated-bf16 cold solves and BF16-inner iterative refinement
on the cantilever presets, against the FP64 answer, through the reference
API (MatFreeOperator(precision="bf16"), solve_equilibrium, solve_refined).
Prints one JSON line per problem."""
from __future__ import annotations

import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_18020_b200 import (CgConfig, MatFreeOperator, SimpParams, build_edof, make_preset,  # noqa: E402
                                   solve_equilibrium, solve_refined)

for scale in [float(eval(a)) for a in (sys.argv[1:] or ["0.2", "1/3", "2/3", "1.0"])]:
    pb = make_preset("cantilever", scale)
    edof = build_edof(pb.mesh)
    rho = np.full(pb.mesh.n_elem, 0.5)
    ops = {p: MatFreeOperator(pb.mesh, edof, pb.bcs, rho, SimpParams(3.0), p) for p in ("fp64", "fp32", "bf16")}
    row = {"mesh": list(pb.mesh.shape) if hasattr(pb.mesh, "shape") else [pb.mesh.nelx, pb.mesh.nely, pb.mesh.nelz],
           "n_elem": pb.mesh.n_elem}
    c64 = None
    for p, op in ops.items():
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        u, rep = solve_equilibrium(op, pb.bcs.force, CgConfig())
        torch.cuda.synchronize()
        if p == "fp64":
            c64 = rep.compliance
        row[p] = {"iterations": rep.iterations, "termination": rep.termination, "compliance": rep.compliance,
                  "compliance_rel_err": abs(rep.compliance - c64) / c64,
                  "verified_rel_residual": rep.verified_rel_residual, "solve_s": time.perf_counter() - t0}
    t0 = time.perf_counter()
    _, ir = solve_refined(ops["fp32"], ops["bf16"], pb.bcs.force)
    row["ir_bf16_inner"] = {"converged": ir.converged, "stagnated": ir.stagnated, "outer_steps": ir.outer_steps,
                            "inner_iterations": ir.inner_iterations, "outer_residuals": ir.outer_residuals,
                            "compliance_rel_err": abs(ir.compliance - c64) / c64,
                            "wall_s": time.perf_counter() - t0}
    print(json.dumps(row), flush=True)
