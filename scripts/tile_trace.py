"""Per-CTA timeline of one cold structured product (TF_TILE_TRACE build).

    make -C paper_2604_18020_b200/csrc OUTDIR=../lib_trace NVEXTRA=-DTF_TILE_TRACE
    TOPOFUSE_B200_LIB=paper_2604_18020_b200/lib_trace/libtopofuse_b200.so \\
        python scripts/tile_trace.py [config] [oz]

Prints the CTA start ramp, the column-setup / prologue / per-layer phase
durations (clock64, converted with the measured clock rate) and the end
spread, from thread 0 of every CTA (k_grid_tile5's TT_* points)."""

from __future__ import annotations

import ctypes
import json
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
if len(sys.argv) > 2:
    os.environ["TF_TILE_OZ"] = sys.argv[2]
os.environ["TF_TILE_AUTOTUNE"] = "0"

import torch  # noqa: E402

from bench import CONFIGS, build_problem  # noqa: E402
from paper_2604_18020_b200 import MatFreeOperator, SimpParams, _lib  # noqa: E402

dims, prec, _ = CONFIGS[cfg]
m, edof, bcs, rho, v = build_problem(dims)
op = MatFreeOperator(m, edof, bcs, rho, SimpParams(3.0), prec)
x = torch.tensor(v.astype(op.precision.dtype), device="cuda")
w = torch.empty_like(x)
oz, ctas = ctypes.c_int32(), ctypes.c_int64()
_lib.call("tf_tile_shape", ctypes.byref(op.dev.grid), 32 if prec == "fp32" else 64, ctypes.byref(oz), ctypes.byref(ctas))
n = ctas.value
buf = torch.zeros(n * 16, dtype=torch.int64, device="cuda")
lib = _lib.load()
lib.tf_tile_trace_set.argtypes = [ctypes.c_void_p]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
out = {}
for rep in range(4):
    for _ in range(3):
        op.apply_device(x, out=w)
    flush.fill_(rep)
    torch.cuda.synchronize()
    assert lib.tf_tile_trace_set(ctypes.c_void_p(buf.data_ptr())) == 0
    op.apply_device(x, out=w)
    torch.cuda.synchronize()
    assert lib.tf_tile_trace_set(ctypes.c_void_p(0)) == 0
    t = buf.view(n, 16).cpu().numpy().astype(np.int64)
    g0, g1 = t[:, 0], t[:, 15]
    clk = t[:, 2:15]
    ghz = float(np.median((t[:, 14] - t[:, 2]) / np.maximum(1, g1 - g0)))
    start = (g0 - g0.min())
    end = (g1 - g0.min())
    ph = lambda a, b: (t[:, b] - t[:, a]) / ghz  # ns
    layers = [ph(4 + k, 5 + k) for k in range(4) if np.all(t[:, 5 + k] > 0)]
    smc = np.bincount(t[:, 1].astype(np.int64))
    rec = {"oz": oz.value, "ctas": n, "clock_ghz": ghz,
           "start_ns": {"p50": float(np.median(start)), "max": float(start.max())},
           "setup_ns": float(np.median(ph(2, 3))), "prologue_ns": float(np.median(ph(3, 4))),
           "layer_ns": [float(np.median(l)) for l in layers],
           "cta_ns": {"p50": float(np.median(ph(2, 14 - 2 + 2))) if False else float(np.median((t[:, 14] - t[:, 2]) / ghz)),
                      "max": float(((t[:, 14] - t[:, 2]) / ghz).max())},
           "end_ns": {"p50": float(np.median(end)), "max": float(end.max())},
           "ctas_per_sm": {"max": int(smc.max()), "min": int(smc[smc > 0].min()), "sms": int((smc > 0).sum())}}
    out[f"rep{rep}"] = rec
    print(json.dumps(rec), flush=True)
Path("gpurun_out").mkdir(exist_ok=True)
Path(f"gpurun_out/tile_trace_{cfg}_{oz.value}.json").write_text(json.dumps(out, indent=1))
