"""A/B of the general-connectivity (edof-reading, red.global) K.v kernels.

    python scripts/edof_ab.py LABEL [configs...]     configs: c2 c5 c2f64 c5f64 (+ _rand: seeded_random)

Per config: mean device time per product (L2 flushed before each step, CUDA
events; the product includes the zeroing of w), GDOF/s, the HBM fraction of
the general-contract compulsory bytes, and the error against the reference's
own apply (tests/golden/hashes_r2.json) where a golden exists."""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from bench import CONFIGS, build_problem, peaks, reference_check  # noqa: E402
from paper_2604_18020_b200 import MatFreeOperator, SimpParams  # noqa: E402
from paper_2604_18020_b200.mesh import BoundaryConditions  # noqa: E402
from paper_2604_18020_b200.operator import compulsory_bytes  # noqa: E402

label = sys.argv[1]
names = sys.argv[2:] or ["c2", "c5", "c2f64", "c5f64", "c2_rand", "c5_rand"]
hbm = peaks()[0]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
out = {}
for name in names:
    cfg = name.replace("_rand", "")
    dims, prec, _ = CONFIGS[cfg]
    m, edof, bcs, rho, v = build_problem(dims)
    perm = None
    if name.endswith("_rand"):
        perm = np.random.default_rng(42).permutation(m.n_dof).astype(np.int32)
        edof = np.ascontiguousarray(perm[edof])
        f = np.zeros(m.n_dof)
        f[perm] = bcs.force
        bcs = BoundaryConditions(np.sort(perm[bcs.fixed_dofs]).astype(np.int64), f)
        vp = np.empty_like(v)
        vp[perm] = v
        v = vp
    op = MatFreeOperator(m, edof, bcs, rho, SimpParams(3.0), prec, grid_kernel="edof", scatter="parallel_atomic")
    x = torch.tensor(v.astype(op.precision.dtype), device="cuda")
    w = torch.empty_like(x)
    for _ in range(5):
        op.apply_device(x, out=w)
    steps = 100
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for a, b in ev:
        flush.fill_(1)
        a.record()
        op.apply_device(x, out=w)
        b.record()
    torch.cuda.synchronize()
    ms = float(np.mean([a.elapsed_time(b) for a, b in ev]))
    byts = compulsory_bytes(m.n_elem, m.n_dof, prec, False)
    out[name] = {"us": 1e3 * ms, "GDOF_s": m.n_dof / ms / 1e6, "hbm_frac": byts / (ms * 1e-3) / 1e9 / hbm,
                 "vs_reference": reference_check(cfg, prec, w.double().cpu().numpy(), perm)}
    print(label, name, json.dumps(out[name]), flush=True)
    del op, x, w
Path("gpurun_out").mkdir(exist_ok=True)
Path(f"gpurun_out/edof_ab_{label}.json").write_text(json.dumps(out, indent=1))
