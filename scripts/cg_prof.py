"""One short FP32/FP64 cold solve for ncu launch lists of a PCG iteration
(run with TF_PCG_NOGRAPH=1 so the iteration's kernels launch outside the
graph):  python scripts/cg_prof.py SCALE fp32|fp64 [max_iter, default 12]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import sys, numpy as np
from paper_2604_18020_b200 import *
scale = float(sys.argv[1]); prec = sys.argv[2]
pb = make_preset('cantilever', scale)
op = MatFreeOperator(pb.mesh, build_edof(pb.mesh), pb.bcs, np.full(pb.mesh.n_elem, 0.5), SimpParams(3.0), prec)
u, rep = solve_equilibrium(op, pb.bcs.force, CgConfig(max_iter=int(sys.argv[3]) if len(sys.argv) > 3 else 12))
print(rep.iterations)
