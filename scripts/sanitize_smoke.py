"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck):
structured tile + pull + exact matvecs, general-edof atomic + coloured, three-stage,
Jacobi, energies, a device PCG (graph + direct mode) and two device SIMP iterations."""
import os

import numpy as np

from paper_2604_18020_b200 import (BoundaryConditions, CgConfig, MatFreeOperator, SimpConfig,
                                   SimpParams, build_edof, make_preset, run_simp, solve_equilibrium)
from paper_2604_18020_b200.mesh import StructuredMesh, cantilever_bcs
from paper_2604_18020_b200.simp import ContinuationSchedule, Phase

m = StructuredMesh(33, 9, 5)
edof = build_edof(m)
bcs = cantilever_bcs(m)
rng = np.random.default_rng(0)
rho = rng.uniform(0.1, 1.0, m.n_elem)
v = rng.standard_normal(m.n_dof)
for prec in ("fp32", "fp64"):
    for kern in ("tile", "pull", "exact"):
        op = MatFreeOperator(m, edof, bcs, rho, SimpParams(3.0), prec, grid_kernel=kern)
        op.apply(v.astype(op.precision.dtype))
    op.diagonal()
    op.element_energies(v)
    for scatter in ("parallel_atomic", "serial"):
        perm = rng.permutation(m.n_dof).astype(np.int32)
        ep = np.ascontiguousarray(perm[edof])
        bp = BoundaryConditions(np.sort(perm[bcs.fixed_dofs]), np.zeros(m.n_dof))
        MatFreeOperator(m, ep, bp, rho, SimpParams(3.0), prec, scatter=scatter).apply(v.astype(op.precision.dtype))
    MatFreeOperator(m, edof, bcs, rho, SimpParams(3.0), prec, variant="three_stage").apply(v.astype(op.precision.dtype))
pb = make_preset("cantilever", 0.2)
for fused in ("1", "0"):
    os.environ["TF_PCG_FUSED"] = fused
    pbm = make_preset("cantilever", 0.2)
    op = MatFreeOperator(pbm.mesh, build_edof(pbm.mesh), pbm.bcs, np.full(pbm.mesh.n_elem, 0.5),
                         SimpParams(3.0), "fp32")
    solve_equilibrium(op, pbm.bcs.force, CgConfig(max_iter=60))
sched = ContinuationSchedule((Phase(1, 2, p=3.0, beta=1.0, move=0.2, rmin_end=1.5),), 1.5)
run_simp(pb, SimpConfig(schedule=sched, precision="fp64"))
print("sanitize workload done")
