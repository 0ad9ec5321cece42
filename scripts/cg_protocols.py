"""Time cold PCG solves per device protocol (resident / fused_graph / graph).

usage: python scripts/cg_protocols.py [preset:scale:prec ...]
Prints one JSON line per (problem, protocol): iterations, termination,
solve ms (CUDA events around tf_pcg_solve, device-resident inputs), us/iteration.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2604_18020_b200 import CgConfig, MatFreeOperator, SimpParams, build_edof, make_preset  # noqa: E402
from paper_2604_18020_b200.mesh import StructuredMesh, cantilever_bcs  # noqa: E402
from paper_2604_18020_b200.solver import device_pcg, pcg_protocol  # noqa: E402

PROTOS = {"resident": {"TF_PCG_RESIDENT": "1"},
          "fused_graph": {"TF_PCG_RESIDENT": "0", "TF_PCG_FUSED": "1"},
          "graph": {"TF_PCG_RESIDENT": "0", "TF_PCG_FUSED": "0"}}


def problem(spec):
    name, scale, prec = spec.split(":")
    if name == "c1":
        m = StructuredMesh(48, 24, 24)
        bcs = cantilever_bcs(m)
    else:
        pb = make_preset(name, float(eval(scale)))
        m, bcs = pb.mesh, pb.bcs
    op = MatFreeOperator(m, build_edof(m), bcs, np.full(m.n_elem, 0.5), SimpParams(3.0), prec)
    return op, bcs


def main():
    specs = sys.argv[1:] or ["c1:1:fp64", "cantilever:1:fp32", "cantilever:1:fp64", "torsion:1:fp64"]
    for spec in specs:
        op, bcs = problem(spec)
        b = torch.as_tensor(bcs.force.astype(op.precision.dtype), device="cuda")
        d = torch.as_tensor(op.diagonal(), device="cuda")
        for proto, env in PROTOS.items():
            os.environ.pop("TF_PCG_RESIDENT", None)
            os.environ.pop("TF_PCG_FUSED", None)
            os.environ.update(env)
            got = pcg_protocol(op)
            if got != proto:
                print(json.dumps({"problem": spec, "protocol": proto, "skipped": f"runs {got}"}))
                continue
            device_pcg(op, b, d, CgConfig(), return_device=True)  # warm-up
            ts = []
            for _ in range(3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                x, rep = device_pcg(op, b, d, CgConfig(), return_device=True)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ms = min(ts)
            c = float(torch.dot(b.double(), x.double()))
            print(json.dumps({"problem": spec, "protocol": proto, "n_elem": op.mesh.n_elem,
                              "iterations": rep.iterations, "termination": rep.termination,
                              "compliance": c, "solve_ms": ms,
                              "us_per_iteration": 1e3 * ms / max(rep.iterations, 1)}), flush=True)


if __name__ == "__main__":
    main()
