"""Density snapshot format of the reference (io.py:104-139), for parity artifacts.

`<base>.bin` holds raw little-endian float64 densities in x-fastest element
order; `<base>.json` is the sidecar {"count", "dims", "dtype", "order"}.
Kept byte-compatible so designs produced on B200 load in the reference tools
and vice versa.
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

DENSITY_ORDER = "x-fastest"  # element = ix + iy*nelx + iz*nelx*nely


def write_density(path_base, rho, dims) -> tuple[Path, Path]:
    nx, ny, nz = (int(d) for d in dims)
    arr = np.ascontiguousarray(rho, dtype=np.float64)
    if arr.size != nx * ny * nz:
        raise ValueError(f"density size {arr.size} != {nx}*{ny}*{nz}")
    base = Path(path_base)
    base.parent.mkdir(parents=True, exist_ok=True)
    bin_path, side_path = base.with_suffix(".bin"), base.with_suffix(".json")
    arr.astype("<f8", copy=False).tofile(bin_path)
    meta = {"count": int(arr.size), "dims": [nx, ny, nz], "dtype": "float64", "order": DENSITY_ORDER}
    side_path.write_text(json.dumps(meta, indent=2, sort_keys=True) + "\n")
    return bin_path, side_path


def read_density(path_base) -> tuple[np.ndarray, tuple[int, int, int]]:
    base = Path(path_base)
    meta = json.loads(base.with_suffix(".json").read_text())
    if meta.get("order") != DENSITY_ORDER or meta.get("dtype") != "float64":
        raise ValueError(f"unsupported density snapshot layout: {meta}")
    rho = np.fromfile(base.with_suffix(".bin"), dtype="<f8")
    dims = tuple(int(d) for d in meta["dims"])
    if rho.size != meta["count"] or rho.size != dims[0] * dims[1] * dims[2]:
        raise ValueError("density snapshot does not match its sidecar")
    return rho, dims
