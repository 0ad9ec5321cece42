"""Warm per-kernel device time of a device PCG solve (torch.profiler/CUPTI):
usage: python scripts/cg_kernel_times.py <cantilever scale> <prec> [iters]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2604_18020_b200 import CgConfig, MatFreeOperator, SimpParams, build_edof, make_preset  # noqa: E402
from paper_2604_18020_b200.solver import device_pcg, pcg_protocol  # noqa: E402

scale, prec = float(eval(sys.argv[1])), sys.argv[2]
its = int(sys.argv[3]) if len(sys.argv) > 3 else 200
pb = make_preset("cantilever", scale)
op = MatFreeOperator(pb.mesh, build_edof(pb.mesh), pb.bcs, np.full(pb.mesh.n_elem, 0.5), SimpParams(3.0), prec)
b = torch.as_tensor(pb.bcs.force.astype(op.precision.dtype), device="cuda")
d = torch.as_tensor(op.diagonal(), device="cuda")
cfg = CgConfig(max_iter=its, recompute_every=0)
device_pcg(op, b, d, cfg, return_device=True)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    x, rep = device_pcg(op, b, d, cfg, return_device=True)
    torch.cuda.synchronize()
tot = {}
for e in prof.events():
    if e.device_type.name == "CUDA":
        k = e.name[:90]
        n, t = tot.get(k, (0, 0.0))
        tot[k] = (n + 1, t + e.device_time)
print("protocol", pcg_protocol(op), "iterations", rep.iterations)
for k, (n, t) in sorted(tot.items(), key=lambda kv: -kv[1][1])[:12]:
    print(f"{t / rep.iterations:9.2f} us/it  {n:6d}x  {t / n:8.2f} us  {k}")
