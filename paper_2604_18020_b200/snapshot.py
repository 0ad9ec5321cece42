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


# -- text reports (io.py:18-104, cli.py:54-67, 224-291) --------------------------------
# 9 significant digits everywhere, so a parse/emit cycle is a fixed point.

FLOAT_FMT = "%.9g"

HISTORY_COLUMNS = ["iteration", "compliance", "grayness", "volume", "cg_iterations", "cg_converged",
                   "p", "beta", "move", "rmin", "restarted", "wall_s"]


def format_float(x) -> str:
    return FLOAT_FMT % float(x)


def format_value(v) -> str:
    """One CSV cell (io.py:25-33): bools as True/False, ints verbatim, floats at 9 digits."""
    if isinstance(v, (bool, np.bool_)):
        return str(bool(v))
    if isinstance(v, (int, np.integer)):
        return str(int(v))
    if isinstance(v, (float, np.floating)):
        return format_float(v)
    return str(v)


def write_csv(path, columns, rows) -> Path:
    """Rows are dicts keyed by column; CRLF-free csv module dialect like io.py:52-60."""
    import csv

    path = Path(path)
    path.parent.mkdir(parents=True, exist_ok=True)
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(columns)
        for row in rows:
            w.writerow([format_value(row.get(c, "")) for c in columns])
    return path


def jsonable(obj):
    """JSON-safe values with floats rounded to 9 significant digits (io.py:71-85)."""
    if isinstance(obj, dict):
        return {str(k): jsonable(v) for k, v in obj.items()}
    if isinstance(obj, (list, tuple)):
        return [jsonable(v) for v in obj]
    if isinstance(obj, np.ndarray):
        return [jsonable(v) for v in obj.tolist()]
    if isinstance(obj, (bool, np.bool_)):
        return bool(obj)
    if isinstance(obj, (int, np.integer)):
        return int(obj)
    if isinstance(obj, (float, np.floating)):
        return float(format_float(obj))
    return obj


def write_json(path, obj) -> Path:
    path = Path(path)
    path.parent.mkdir(parents=True, exist_ok=True)
    path.write_text(json.dumps(jsonable(obj), indent=2, sort_keys=True) + "\n")
    return path


def write_residual_history(path, history) -> Path:
    rows = [{"iteration": i, "rel_residual": float(r)} for i, r in enumerate(history)]
    return write_csv(path, ["iteration", "rel_residual"], rows)


def history_rows(result) -> list[dict]:
    from dataclasses import asdict

    return [asdict(rec) for rec in result.history]


def solve_record(report, mesh, preset, scale, scatter, backend="b200") -> dict:
    """The reference's solve payload (cli.py:224-241)."""
    return {"preset": preset, "scale": scale, "n_elem": mesh.n_elem, "n_dof": mesh.n_dof,
            "scatter": scatter, "backend": backend, "converged": report.converged,
            "termination": report.termination, "iterations": report.iterations,
            "rel_residual": report.rel_residual, "verified_rel_residual": report.verified_rel_residual,
            "compliance": report.compliance, "matvecs": report.matvecs, "wall_time_s": report.wall_time,
            "precision": report.precision, "variant": report.variant}


def simp_summary(result, problem, precision, variant, scatter, iters, cg_cap, seed) -> dict:
    """The reference's SIMP summary payload (cli.py:268-290)."""
    sel = result.selected
    return {
        "preset": problem.name, "scale": problem.scale,
        "dims": [problem.mesh.nelx, problem.mesh.nely, problem.mesh.nelz],
        "volume_fraction": problem.volume_fraction, "precision": precision, "variant": variant,
        "scatter": scatter, "iters": iters, "cg_cap": cg_cap, "seed": seed,
        "selected": None if sel is None else {"iteration": sel.iteration, "compliance": sel.compliance,
                                              "grayness": sel.grayness, "p": sel.p, "beta": sel.beta},
        "restart_count": result.restart_count, "total_cg_iterations": result.total_cg_iterations,
        "wall_s": result.wall_s, "history": history_rows(result),
    }


def write_simp_artifacts(out_dir, result, problem, precision="fp64", variant="fused", scatter="serial",
                         iters=None, cg_cap=1000, seed=42) -> dict:
    """`<out>/simp_<preset>_<prec>_history.csv`, `_summary.json` and the selected
    density snapshot, named and laid out as cmd_simp writes them (cli.py:250-297)."""
    out = Path(out_dir)
    stem = f"simp_{problem.name}_{precision}"
    iters = iters if iters is not None else len(result.history)
    paths = {"history": write_csv(out / f"{stem}_history.csv", HISTORY_COLUMNS, history_rows(result)),
             "summary": write_json(out / f"{stem}_summary.json",
                                   simp_summary(result, problem, precision, variant, scatter, iters, cg_cap,
                                                seed))}
    if result.selected is not None:
        dims = (problem.mesh.nelx, problem.mesh.nely, problem.mesh.nelz)
        paths["density"] = write_density(out / f"{stem}_selected", result.selected.rho_phys, dims)[0]
    return paths
