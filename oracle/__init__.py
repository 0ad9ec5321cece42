"""TEST INFRASTRUCTURE ONLY -- the CPU oracle (checker) for the B200 hot path.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) may import this package.  The product package
``paper_2604_18020_b200`` never imports it; a product call that ends up here
would void every parity claim.

Contents
  * ctypes bindings to ``lib/libtopofuse_oracle.so`` -- a plain-C restatement
    of the reference numba element loops (see topofuse_oracle.c for the
    file:line map and the floating-point order it reproduces);
  * numpy restatements of the reference operator glue (masking, fixed-DOF
    pass-through, Jacobi diagonal) and of the Jacobi-PCG recurrence.

Pinning: tests/test_oracle.py checks these functions bitwise against golden
outputs of the real reference (tests/golden/*.npz, produced by
tests/golden/make_golden.py importing /root/reference/pkg/src).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "lib" / "libtopofuse_oracle.so"
_lib = None

_I32P = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_F64P = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_F32P = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_I64 = ctypes.c_int64


def build(force: bool = False) -> Path:
    """Compile the oracle C library with its Makefile (gcc, -ffp-contract=off)."""
    if force or not _LIB_PATH.exists() or (
        _LIB_PATH.stat().st_mtime < (_HERE / "topofuse_oracle.c").stat().st_mtime
    ):
        subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(_LIB_PATH))
        for prec, P in (("f64", _F64P), ("f32", _F32P)):
            for name in ("orc_fused_serial_", "orc_fused_atomic_"):
                fn = getattr(L, name + prec)
                fn.argtypes = [_I32P, P, P, P, P, _I64]
                fn.restype = None
            g = getattr(L, "orc_gather_" + prec)
            g.argtypes = [_I32P, P, P, _I64]
            g.restype = None
            m = getattr(L, "orc_gemm_" + prec)
            m.argtypes = [P, P, P, P, _I64]
            m.restype = None
            j = getattr(L, "orc_jacobi_" + prec)
            j.argtypes = [_I32P, P, P, _F64P, _I64]
            j.restype = None
        L.orc_scatter_f64.argtypes = [_I32P, _F64P, _F64P, _I64]
        L.orc_scatter_f32_into_f64.argtypes = [_I32P, _F32P, _F64P, _I64]
        L.orc_element_energies.argtypes = [_I32P, _F64P, _F64P, _F64P, _I64]
        L.orc_fused_serial_bf16.argtypes = [_I32P, _F32P, _F32P, _F32P, _F32P, _I64]
        L.orc_gemm_bf16.argtypes = [_F32P, _F32P, _F32P, _F32P, _I64]
        L.orc_jacobi_bf16.argtypes = [_I32P, _F32P, _F32P, _F32P, _I64]
        L.orc_round_bf16.argtypes = [_F32P, _F32P, _I64]
        for f in ("orc_fused_serial_bf16", "orc_gemm_bf16", "orc_jacobi_bf16", "orc_round_bf16"):
            getattr(L, f).restype = None
        L.orc_num_threads.restype = ctypes.c_int
        L.orc_set_num_threads.argtypes = [ctypes.c_int]
        _lib = L
    return _lib


def _tag(dtype) -> str:
    dt = np.dtype(dtype)
    if dt == np.float64:
        return "f64"
    if dt == np.float32:
        return "f32"
    raise TypeError(f"oracle supports float32/float64, got {dt}")


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


# -- kernel-contract restatements (signatures of _kernels_numba.py) ------------


def fused_serial(edof, ke, scale, v, out) -> None:
    """_kernels_numba.py:146-162 -- accumulate into `out` (caller-zeroed)."""
    t = _tag(v.dtype)
    dt = v.dtype
    getattr(lib(), "orc_fused_serial_" + t)(
        _c(edof, np.int32), _c(ke, dt), _c(scale, dt), _c(v, dt), out, edof.shape[0]
    )


def fused_atomic(edof, ke, scale, v, out, threads: int | None = None) -> None:
    """_kernels_numba.py:183-196 -- OpenMP + atomics, nondeterministic order."""
    t = _tag(v.dtype)
    dt = v.dtype
    if threads:
        lib().orc_set_num_threads(int(threads))
    getattr(lib(), "orc_fused_atomic_" + t)(
        _c(edof, np.int32), _c(ke, dt), _c(scale, dt), _c(v, dt), out, edof.shape[0]
    )


def gather(edof, v):
    """_kernels_numba.py:82-92."""
    u = np.empty((edof.shape[0], 24), dtype=v.dtype)
    getattr(lib(), "orc_gather_" + _tag(v.dtype))(_c(edof, np.int32), _c(v, v.dtype), u, edof.shape[0])
    return u


def gemm(u_elem, ke, scale):
    """_kernels_numba.py:95-109 (scale applied after the row sum)."""
    dt = u_elem.dtype
    f = np.empty_like(u_elem)
    getattr(lib(), "orc_gemm_" + _tag(dt))(
        _c(u_elem, dt), _c(ke, dt), _c(scale, dt), f, u_elem.shape[0]
    )
    return f


def scatter_serial(edof, f_elem, acc) -> None:
    """_kernels_numba.py:129-133 with `acc` float64."""
    if f_elem.dtype == np.float64:
        lib().orc_scatter_f64(_c(edof, np.int32), _c(f_elem, np.float64), acc, edof.shape[0])
    else:
        lib().orc_scatter_f32_into_f64(_c(edof, np.int32), _c(f_elem, np.float32), acc, edof.shape[0])


def jacobi_diag(edof, ke_diag, scale, out) -> None:
    """_kernels_numba.py:217-226; `out` is float64."""
    dt = scale.dtype
    getattr(lib(), "orc_jacobi_" + _tag(dt))(
        _c(edof, np.int32), _c(ke_diag, dt), _c(scale, dt), out, edof.shape[0]
    )


def element_energies(edof, ke, u):
    """_kernels_numba.py:241-256, FP64."""
    out = np.empty(edof.shape[0], dtype=np.float64)
    lib().orc_element_energies(
        _c(edof, np.int32), _c(ke, np.float64), _c(u, np.float64), out, edof.shape[0]
    )
    return out


def round_bf16(x):
    """precision.py:65-85 round_to_bf16 (float32 in, float32 out)."""
    x = _c(x, np.float32)
    y = np.empty_like(x)
    lib().orc_round_bf16(x, y, x.size)
    return y


def fused_serial_bf16(edof, ke, scale, v, out) -> None:
    """_kernels_numba.py:166-180 -- v pre-quantized, out float32 accumulated."""
    lib().orc_fused_serial_bf16(_c(edof, np.int32), _c(ke, np.float32), _c(scale, np.float32),
                                _c(v, np.float32), out, edof.shape[0])


def gemm_bf16(u_elem, ke, scale):
    """_kernels_numba.py:113-126."""
    f = np.empty((u_elem.shape[0], 24), dtype=np.float32)
    lib().orc_gemm_bf16(_c(u_elem, np.float32), _c(ke, np.float32), _c(scale, np.float32), f,
                        u_elem.shape[0])
    return f


def jacobi_diag_bf16(edof, ke_diag, scale, out) -> None:
    """_kernels_numba.py:230-238; `out` float32."""
    lib().orc_jacobi_bf16(_c(edof, np.int32), _c(ke_diag, np.float32), _c(scale, np.float32), out,
                          edof.shape[0])


def apply_bf16(edof, ke, scale, v, fixed_dofs, n_dof, variant="fused"):
    """MatFreeOperator.apply for precision "bf16" (operator.py:83-117):
    masked input rounded to bf16, bf16 kernels, pass-through of the raw v."""
    free = np.ones(n_dof, dtype=bool)
    free[fixed_dofs] = False
    x = round_bf16(np.where(free, np.asarray(v, dtype=np.float32), 0).astype(np.float32))
    out = np.zeros(n_dof, dtype=np.float32)
    if variant == "fused":
        fused_serial_bf16(edof, ke, scale, x, out)
    else:
        f = gemm_bf16(gather(edof, x), ke, scale)
        acc = np.zeros(n_dof)
        scatter_serial(edof, f, acc)
        out[:] = acc
    out[fixed_dofs] = np.asarray(v, dtype=np.float32)[fixed_dofs]
    return out


def diagonal_bf16(edof, ke, scale, fixed_dofs, n_dof):
    """MatFreeOperator.diagonal for bf16 (operator.py:122-126)."""
    out = np.zeros(n_dof, dtype=np.float32)
    jacobi_diag_bf16(edof, np.diag(ke).copy(), scale, out)
    out[fixed_dofs] = 1.0
    return out


# -- operator glue (operator.py:83-132) -----------------------------------------


def apply(edof, ke, scale, v, fixed_dofs, n_dof, variant="fused", scatter="serial"):
    """MatFreeOperator.apply restated (operator.py:90-117) for fp32/fp64.

    `ke`/`scale` are already in the working dtype; v is cast to it.
    """
    dt = np.asarray(ke).dtype
    free = np.ones(n_dof, dtype=bool)
    free[np.asarray(fixed_dofs, dtype=np.int64)] = False
    x = np.ascontiguousarray(np.where(free, np.asarray(v, dtype=dt), 0), dtype=dt)
    out = np.zeros(n_dof, dtype=dt)
    if variant == "fused":
        (fused_serial if scatter == "serial" else fused_atomic)(edof, ke, scale, x, out)
    else:
        u_elem = gather(edof, x)
        f_elem = gemm(u_elem, ke, scale)
        acc = np.zeros(n_dof, dtype=np.float64)
        scatter_serial(edof, f_elem, acc)
        out[:] = acc
    out[fixed_dofs] = np.asarray(v, dtype=dt)[fixed_dofs]
    return out


def diagonal(edof, ke, scale, fixed_dofs, n_dof):
    """MatFreeOperator.diagonal (operator.py:122-132), fp32/fp64."""
    dt = np.asarray(ke).dtype
    acc = np.zeros(n_dof, dtype=np.float64)
    jacobi_diag(edof, np.diag(ke).copy(), np.asarray(scale, dtype=dt), acc)
    out = acc.astype(dt)
    out[fixed_dofs] = 1.0
    return out


# -- Jacobi-PCG recurrence (solver.py:57-147) -----------------------------------


def pcg(apply_op, b, diag, rel_tol=1e-5, max_iter=1000, recompute_every=50, x0=None,
        quantize_krylov=False):
    """Restatement of the reference pcg.  Returns (x, info dict).

    Same recurrence, stop rule, refresh period, breakdown and divergence
    semantics; vectors stay in b's dtype and dots are numpy dots in that
    dtype, exactly as the reference computes them.
    """
    b = np.ascontiguousarray(b)
    bnorm = float(np.linalg.norm(b))
    if bnorm == 0.0:
        return np.zeros_like(b), dict(iterations=0, termination="converged", rel=0.0,
                                      history=[0.0], matvecs=0)
    matvecs = 0
    if x0 is None:
        x = np.zeros_like(b)
        r = b.copy()
    else:
        x = np.array(x0, dtype=b.dtype, copy=True)
        r = b - apply_op(x)
        matvecs += 1
    inv_diag = 1.0 / np.asarray(diag, dtype=b.dtype)
    z = r * inv_diag
    p = z.copy()
    rz = float(np.dot(r, z))
    rel = float(np.linalg.norm(r)) / bnorm
    hist = [rel]
    term = "converged" if rel <= rel_tol else "max_iter"
    done = rel <= rel_tol
    it = 0
    while not done and it < max_iter:
        it += 1
        q = apply_op(p)
        matvecs += 1
        pq = float(np.dot(p, q))
        if not (math.isfinite(pq) and math.isfinite(rz)):
            raise FloatingPointError(f"CG diverged at iteration {it}")
        if pq <= 0.0:
            term = "breakdown"
            break
        alpha = rz / pq
        x += alpha * p
        if recompute_every and it % recompute_every == 0:
            r = b - apply_op(x)
            matvecs += 1
        else:
            r -= alpha * q
        rn = float(np.linalg.norm(r))
        if not math.isfinite(rn):
            raise FloatingPointError(f"CG diverged at iteration {it}")
        rel = rn / bnorm
        hist.append(rel)
        if rel <= rel_tol:
            term = "converged"
            break
        z = r * inv_diag
        rz_new = float(np.dot(r, z))
        p = z + (rz_new / rz) * p
        if quantize_krylov:  # solver.py:134-136
            p = round_bf16(p)
            r = round_bf16(r)
        rz = rz_new
    return x, dict(iterations=it, termination=term, rel=rel, history=hist, matvecs=matvecs)


def threads() -> int:
    return int(lib().orc_num_threads())


def set_threads(n: int) -> None:
    lib().orc_set_num_threads(int(n))


def default_threads() -> int:
    return os.cpu_count() or 1
