"""ctypes binding of libtopofuse_b200.so (the C ABI in include/topofuse_b200.h).

The product path has no CPU fallback: if the library is missing or no CUDA
device is present, every compute entry point raises.  Device buffers are
torch CUDA tensors; only their data pointers cross the boundary.
"""

from __future__ import annotations

import ctypes
import os
import re
import subprocess
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("TOPOFUSE_B200_LIB", _PKG / "lib" / "libtopofuse_b200.so"))
HEADER = _PKG.parent / "include" / "topofuse_b200.h"
CSRC = _PKG / "csrc"

TF_OK = 0
TF_ERR_UNSUPPORTED = 3
TF_OC_MAX_LAMS = 15
TF_ACCUMULATE = 1
TF_MASK_INPUT = 2
TF_PASS_FIXED = 4
TF_GRID_FAST = 0
TF_GRID_BITWISE = 1
TF_GRID_PULL = 2
TF_SCATTER_ATOMIC = 0
TF_SCATTER_COLORED = 1
TERMINATIONS = ("converged", "max_iter", "breakdown", "diverged")


class TfError(RuntimeError):
    pass


class tf_grid(ctypes.Structure):
    _fields_ = [("nelx", ctypes.c_int32), ("nely", ctypes.c_int32), ("nelz", ctypes.c_int32)]


class tf_slab_desc(ctypes.Structure):
    _fields_ = [
        ("grid", tf_grid),
        ("precision", ctypes.c_int32),
        ("ke", ctypes.c_void_p),
        ("scale", ctypes.c_void_p),
        ("node_fixed", ctypes.c_void_p),
        ("fixed", ctypes.c_void_p),
        ("n_fixed", ctypes.c_int64),
        ("owned", ctypes.c_void_p),
        ("left_idx", ctypes.c_void_p),
        ("right_idx", ctypes.c_void_p),
        ("plane_len", ctypes.c_int64),
        ("has_left", ctypes.c_int32),
        ("has_right", ctypes.c_int32),
        ("rank", ctypes.c_int32),
        ("world", ctypes.c_int32),
        ("peer_base", ctypes.c_void_p),
        ("off_planes", ctypes.c_int64),
        ("plane_bytes", ctypes.c_int64),
        ("off_flags", ctypes.c_int64),
        ("off_arflags", ctypes.c_int64),
        ("off_slots", ctypes.c_int64),
        ("max_scalars", ctypes.c_int64),
        ("bl", ctypes.c_int32),
        ("br", ctypes.c_int32),
    ]


class tf_pcg_desc(ctypes.Structure):
    _fields_ = [
        ("precision", ctypes.c_int),
        ("structured", ctypes.c_int),
        ("grid", tf_grid),
        ("edof", ctypes.c_void_p),
        ("n_elem", ctypes.c_int64),
        ("n_dof", ctypes.c_int64),
        ("ke", ctypes.c_void_p),
        ("node_fixed", ctypes.c_void_p),
        ("fixed", ctypes.c_void_p),
        ("n_fixed", ctypes.c_int64),
        ("grid_variant", ctypes.c_int),
        ("flags", ctypes.c_int),
    ]


class tf_oc_report(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("evaluations", ctypes.c_int32),
                ("lam", ctypes.c_double), ("best_err", ctypes.c_double)]


OC_STATUS = ("ok", "saturated", "stalled", "bad_input")


class tf_pcg_report(ctypes.Structure):
    _fields_ = [
        ("iterations", ctypes.c_int32),
        ("termination", ctypes.c_int32),
        ("matvecs", ctypes.c_int32),
        ("_pad", ctypes.c_int32),
        ("rel_residual", ctypes.c_double),
    ]


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_U32 = ctypes.c_uint32
_INT = ctypes.c_int

# name -> argtypes (restype int unless noted)
_SIGS = {
    "tf_version": [],
    "tf_device_count": [],
    "tf_build_node_fixed": [_P, _P, _I64, _P, _P],
    "tf_matvec_grid_f32": [_P, _P, _P, _P, _P, _P, _U32, _INT, _P],
    "tf_matvec_grid_f64": [_P, _P, _P, _P, _P, _P, _U32, _INT, _P],
    "tf_matvec_grid_range_f32": [_P, _P, _P, _P, _P, _P, _U32, ctypes.c_int32, ctypes.c_int32, _P],
    "tf_matvec_grid_range_f64": [_P, _P, _P, _P, _P, _P, _U32, ctypes.c_int32, ctypes.c_int32, _P],
    "tf_matvec_edof_f32": [_P, _P, _P, _P, _P, _I64, _INT, _P, _P, _INT, _P],
    "tf_matvec_edof_f64": [_P, _P, _P, _P, _P, _I64, _INT, _P, _P, _INT, _P],
    "tf_edof_merge_mask": [_P, _I64, _I64, _P, _P],
    "tf_matvec_edof_merged_f32": [_P, _P, _P, _P, _P, _P, _I64, _P],
    "tf_matvec_edof_merged_f64": [_P, _P, _P, _P, _P, _P, _I64, _P],
    "tf_pass_fixed_f32": [_P, _I64, _P, _P, _P],
    "tf_pass_fixed_f64": [_P, _I64, _P, _P, _P],
    "tf_gather_f32": [_P, _P, _P, _I64, _P],
    "tf_gather_f64": [_P, _P, _P, _I64, _P],
    "tf_gemm_f32": [_P, _P, _P, _P, _I64, _P],
    "tf_gemm_f64": [_P, _P, _P, _P, _I64, _P],
    "tf_scatter_f32": [_P, _P, _P, _I64, _P],
    "tf_scatter_f64": [_P, _P, _P, _I64, _P],
    "tf_jacobi_grid_f32": [_P, _P, _P, _P, _P, _P, _P],
    "tf_jacobi_grid_f64": [_P, _P, _P, _P, _P, _P, _P],
    "tf_jacobi_edof_f32": [_P, _P, _P, _P, _I64, _P],
    "tf_jacobi_edof_f64": [_P, _P, _P, _P, _I64, _P],
    "tf_energies_grid_f64": [_P, _P, _P, _P, _P],
    "tf_energies_edof_f64": [_P, _P, _P, _P, _I64, _P],
    "tf_pcg_create": [_P, _P, _P],
    "tf_pcg_solve": [_P, _P, _P, _P, _P, _INT, ctypes.c_double, ctypes.c_int32, ctypes.c_int32,
                     _P, _P],
    "tf_pcg_destroy": [_P],
    "tf_pcg_protocol": [_P],
    "tf_pcg_set_quantize_krylov": [_P, _INT],
    "tf_tile_shape": [_P, _INT, _P, _P],
    "tf_edof_csr_build": [_P, _I64, _I64, _P, _P, _P],
    "tf_scatter_pull_f32": [_P, _P, _P, _P, _I64, _P],
    "tf_scatter_pull_f64": [_P, _P, _P, _P, _I64, _P],
    "tf_matvec_edof_pull_bf16": [_P, _P, _P, _P, _P, _I64, _I64, _P, _P, _P, _INT, _P],
    "tf_jacobi_edof_pull_f32": [_P, _P, _P, _P, _P, _I64, _P],
    "tf_jacobi_edof_pull_f64": [_P, _P, _P, _P, _P, _I64, _P],
    "tf_matvec_edof_pull_f32": [_P, _P, _P, _P, _P, _I64, _I64, _P, _P, _P, _INT, _P],
    "tf_matvec_edof_pull_f64": [_P, _P, _P, _P, _P, _I64, _I64, _P, _P, _P, _INT, _P],
    "tf_host_alloc": [_P, ctypes.c_size_t],
    "tf_host_free": [_P],
    "tf_matvec_grid_stream_f32": [_P, _P, _P, _P, _U32, _I64, _P, _P, _P, _P, _P],
    "tf_matvec_grid_stream_f64": [_P, _P, _P, _P, _U32, _I64, _P, _P, _P, _P, _P],
    "tf_matvec_edof_bf16": [_P, _P, _P, _P, _P, _I64, _INT, _P, _P, _INT, _INT, _P],
    "tf_matvec_edof_bf16_f64": [_P, _P, _P, _P, _P, _I64, _P],
    "tf_gemm_bf16": [_P, _P, _P, _P, _I64, _P],
    "tf_jacobi_edof_bf16": [_P, _P, _P, _P, _I64, _P],
    "tf_round_bf16": [_I64, _P, _P, _P],
    "tf_filter_rowsum_f64": [_P, ctypes.c_double, _P, _P],
    "tf_filter_grid_f64": [_P, ctypes.c_double, _P, _P, _P, _INT, _P],
    "tf_project_f64": [_I64, ctypes.c_double, ctypes.c_double, _P, _P, _P, _P],
    "tf_simp_scale_f32": [_I64, ctypes.c_double, ctypes.c_double, _P, _P, _P, _P],
    "tf_simp_scale_f64": [_I64, ctypes.c_double, ctypes.c_double, _P, _P, _P, _P],
    "tf_sensitivity_f64": [_I64, ctypes.c_double, ctypes.c_double, _P, _P, _P, _P, _P],
    "tf_stats_f64": [_I64, _P, _P, _P, _P, _P, _P, _P],
    "tf_oc_update_f64": [_I64, _P, _P, _P, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                         ctypes.c_double, _INT, _P, _P, _P, _P],
    "tf_oc_volumes_f64": [_I64, _P, _P, _P, ctypes.c_double, ctypes.c_double, _P, _INT, _P, _P, _P],
    "tf_oc_apply_f64": [_I64, _P, _P, _P, ctypes.c_double, ctypes.c_double, ctypes.c_double, _P, _P],
    "tf_slab_cg_start": [_P, _P, ctypes.c_double, _INT, _P],
    "tf_peer_alloc": [_P, ctypes.c_size_t],
    "tf_peer_free": [_P],
    "tf_ipc_handle_bytes": [],
    "tf_ipc_export": [_P, _P],
    "tf_ipc_open": [_P, _P],
    "tf_ipc_close": [_P],
    "tf_stream_write_u32": [_P, ctypes.c_uint32, _P],
    "tf_stream_wait_u32": [_P, ctypes.c_uint32, _P],
    "tf_rank_sum_f64": [_P, _INT, _INT, _P, _P],
    "tf_stream_wait_many_u32": [_P, _INT, ctypes.c_uint32, _P],
    "tf_slab_create": [_P, _P],
    "tf_abi_struct_sizes": [_P, _INT],
    "tf_slab_destroy": [_P],
    "tf_slab_apply": [_P, _P, _P, _P, _P],
    "tf_slab_allreduce": [_P, _P, _INT, _P, _P],
    "tf_slab_pcg_iterate": [_P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _INT, _INT, _INT, _P, _INT, _P, _P],
    "tf_slab_pcg_graph": [_P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _INT, _INT, _INT, _P, _INT, _P, _P, _P],
    "tf_slab_take_error": [_P, _P],
}
for _s in ("f32", "f64"):
    _SIGS.update({
        f"tf_slab_dot_{_s}": [_I64, _P, _P, _P, _P, _P, _P],
        f"tf_slab_cg_begin_{_s}": [_I64, _P, _P, _P, _P, _P, _P, _P, _P],
        f"tf_slab_cg_pq_{_s}": [_I64, _P, _P, _P, _P, _P, _P, _P],
        f"tf_slab_cg_alpha_{_s}": [_I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _INT, _P, _P],
        f"tf_slab_cg_residual_{_s}": [_I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P],
        f"tf_slab_cg_beta_{_s}": [_I64, _P, _P, _P, _P, _P, _INT, _P],
        f"tf_plane_put_{_s}": [_P, _P, _I64, _P, _P],
        f"tf_plane_add_{_s}": [_P, _P, _I64, _P, _INT, _P],
        f"tf_put_flags_{_s}": [_P, _P, _P, _P, _INT, _I64, ctypes.c_uint32, _P, _P],
        f"tf_plane_add2_{_s}": [_P, _P, _P, _P, _P, _I64, _P],
        f"tf_jacobi_grid_partial_{_s}": [_P, _P, _P, _P, _P],
    })

_lib = None


def header_symbols() -> list[str]:
    """Every function the C header declares (parsed from include/topofuse_b200.h)."""
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\**\s+\**(tf_\w+)\s*\(", text, re.M)))


def build(verbose: bool = False) -> Path:
    """Compile the sm_100a library in-tree with the csrc Makefile (nvcc)."""
    out = subprocess.run(["make", "-C", str(CSRC), "-j4"], capture_output=True, text=True)
    if out.returncode != 0:
        raise TfError("nvcc build failed:\n" + out.stdout[-4000:] + out.stderr[-4000:])
    if verbose:
        print(out.stdout)
    return LIB_PATH


def load() -> ctypes.CDLL:
    """Load the library (no compute); raises when it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise TfError(f"{LIB_PATH} not built -- run __graft_entry__.build() (no CPU fallback)")
    L = ctypes.CDLL(str(LIB_PATH))
    for name, args in _SIGS.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    L.tf_work_doubles.restype = ctypes.c_int64
    L.tf_work_doubles.argtypes = [ctypes.c_int64]
    L.tf_oc_work_doubles.restype = ctypes.c_int64
    L.tf_oc_work_doubles.argtypes = [ctypes.c_int64]
    L.tf_slab_work_doubles.restype = ctypes.c_int64
    L.tf_slab_work_doubles.argtypes = [ctypes.c_int64]
    L.tf_last_error.restype = ctypes.c_char_p
    L.tf_last_error.argtypes = []
    _lib = L
    return L


def check(rc: int, what: str = "") -> None:
    if rc != TF_OK:
        msg = load().tf_last_error().decode(errors="replace")
        raise TfError(f"{what or 'topofuse_b200'} failed (code {rc}): {msg}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)
