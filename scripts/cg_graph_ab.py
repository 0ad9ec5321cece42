"""Graph-protocol A/B: wall time per CG iteration of cold solves (c4 FP32,
c2 FP64, c5 FP32) at a refresh period of 50 (sparse-refresh graph) and 7
(per-iteration IF node), with the resident protocol switched off; run once
plain and once with TF_PCG_SPARSE_IF=0.  Compliance printed to show the
results are bitwise the same."""
import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2604_18020_b200 import CgConfig, MatFreeOperator, SimpParams, build_edof, make_preset, pcg
from paper_2604_18020_b200.solver import pcg_protocol
os.environ["TF_PCG_RESIDENT"] = "0"
for spec in ["5/3:fp32", "1.0:fp64", "17/6:fp32"]:
    sc, prec = spec.split(":")
    pb = make_preset("cantilever", float(eval(sc)))
    op = MatFreeOperator(pb.mesh, build_edof(pb.mesh), pb.bcs, np.full(pb.mesh.n_elem, 0.5), SimpParams(3.0), prec)
    d = op.diagonal(); b = pb.bcs.force.astype(op.precision.dtype)
    for rec in (50, 7):
        cfg = CgConfig(recompute_every=rec)
        pcg(op, b, d, cfg)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); t = time.perf_counter()
        x, rep = pcg(op, b, d, cfg)
        torch.cuda.synchronize(); dt = time.perf_counter() - t
        print(spec, rec, pcg_protocol(op), rep.iterations, rep.termination, f"{1e6*dt/rep.iterations:.2f} us/it (wall)", f"c={float(pb.bcs.force @ x):.10f}", os.environ.get("TF_PCG_SPARSE_IF"), flush=True)
