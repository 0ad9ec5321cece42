"""A/B of the structured K.v kernels on one GPU (run one variant per process:
the launch-shape autotune cache is per process).

    python scripts/tile_ab.py VARIANT [configs...]     VARIANT: a label | ozN (pinned chunk height)

Per config: mean device time per product with L2 flushed before each step
(bench.py protocol), the tuned launch shape, and the sha256 of the product
(bitwise comparison across variants)."""

from __future__ import annotations

import ctypes
import hashlib
import json
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

variant = sys.argv[1]
# "prod": autotuned z-chunk; "ozN": pinned chunk height; any other name: a
# label for the current build (A/B across builds)
if variant.startswith("oz"):
    os.environ["TF_TILE_OZ"] = variant[2:]

import torch  # noqa: E402

from bench import CONFIGS, build_problem, reference_check  # noqa: E402
from paper_2604_18020_b200 import MatFreeOperator, SimpParams, _lib  # noqa: E402

names = sys.argv[2:] or ["c2", "c3", "c4", "c5", "c2f64", "c5f64"]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
out = {}
for name in names:
    dims, prec, _ = CONFIGS[name]
    m, edof, bcs, rho, v = build_problem(dims)
    op = MatFreeOperator(m, edof, bcs, rho, SimpParams(3.0), prec)
    x = torch.tensor(v.astype(op.precision.dtype), device="cuda")
    w = torch.empty_like(x)
    for _ in range(5):
        op.apply_device(x, out=w)
    torch.cuda.synchronize()
    steps = 200
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for a, b in ev:
        flush.fill_(1)
        a.record()
        op.apply_device(x, out=w)
        b.record()
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) for a, b in ev]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        op.apply_device(x, out=w)
    e1.record()
    torch.cuda.synchronize()
    oz, ctas = ctypes.c_int32(), ctypes.c_int64()
    _lib.call("tf_tile_shape", ctypes.byref(op.dev.grid), 32 if prec == "fp32" else 64, ctypes.byref(oz),
              ctypes.byref(ctas))
    out[name] = {"us_cold": 1e3 * float(np.mean(ms)), "us_cold_min": 1e3 * float(np.min(ms)),
                 "us_warm": 1e3 * e0.elapsed_time(e1) / steps, "oz": oz.value, "ctas": ctas.value,
                 "sha": hashlib.sha256(w.cpu().numpy().tobytes()).hexdigest()[:16],
                 "vs_reference": reference_check(name, prec, w.double().cpu().numpy())}
    print(variant, name, json.dumps(out[name]), flush=True)
Path("gpurun_out").mkdir(exist_ok=True)
Path(f"gpurun_out/tile_ab_{variant}.json").write_text(json.dumps(out, indent=1))
