"""The reference kernel-module contract, served by the B200 library.

Same functions and signatures as reference _kernels_numba.py / _kernels_numpy.py
(see backend.py:38-46): a caller that resolves its kernel module through
``get_backend()`` can be pointed at this module instead (INTEGRATION.md shows
the one-line registration).  Arguments are host numpy arrays as in the
reference; each call stages them on the current CUDA device, runs the
sm_100a kernel and writes results back in place.  ``out``/``acc`` are
accumulated into, exactly like the reference.
"""

from __future__ import annotations

import numpy as np

from . import _device as D
from . import _lib

PARALLEL = True  # atomic modes run many-threaded (one GPU thread per element)


def _sfx(a):
    return "f64" if np.asarray(a).dtype == np.float64 else "f32"


def _fused(edof, ke, scale, v, out, mode):
    dt = np.asarray(v).dtype
    edof = np.ascontiguousarray(edof, dtype=np.int32)
    e_d = D.to_dev(edof, np.int32)
    s_d = D.to_dev(scale, dt)
    v_d = D.to_dev(v, dt)
    o_d = D.to_dev(out, dt)
    ke_h = np.ascontiguousarray(ke, dtype=dt)
    if mode == _lib.TF_SCATTER_COLORED:
        from .mesh import StructuredMesh
        from .operator import element_colouring

        # contract gives no mesh: colour greedily on the connectivity itself
        n = edof.shape[0]
        order, offsets = element_colouring(StructuredMesh(n, 1, 1), edof)
        o_ = D.to_dev(order, np.int32)
        _lib.call(f"tf_matvec_edof_{_sfx(v)}", D.ptr(e_d), ke_h.ctypes.data, D.ptr(s_d), D.ptr(v_d),
                  D.ptr(o_d), n, mode, D.ptr(o_), offsets.ctypes.data, len(offsets) - 1,
                  D.stream_ptr())
    else:
        _lib.call(f"tf_matvec_edof_{_sfx(v)}", D.ptr(e_d), ke_h.ctypes.data, D.ptr(s_d), D.ptr(v_d),
                  D.ptr(o_d), edof.shape[0], mode, None, None, 0, D.stream_ptr())
    out[...] = o_d.cpu().numpy()


def fused_serial(edof, ke, scale, v, out) -> None:
    """fused K v accumulated into out in the reference's element order --
    bitwise _kernels_numba.py:146-162 (row sums + ascending-element pull)."""
    t = D.torch()
    dt = np.asarray(v).dtype
    edof = np.ascontiguousarray(edof, dtype=np.int32)
    n_elem, n_dof = edof.shape[0], out.shape[0]
    e_d = D.to_dev(edof, np.int32)
    s_d = D.to_dev(scale, dt)
    v_d = D.to_dev(v, dt)
    o_d = D.to_dev(out, dt)
    off, ent = _csr(e_d, n_elem, n_dof)
    rows = t.empty(n_elem * 24, dtype=t.float64, device=e_d.device)
    ke_h = np.ascontiguousarray(ke, dtype=dt)
    _lib.call(f"tf_matvec_edof_pull_{_sfx(v)}", D.ptr(e_d), ke_h.ctypes.data, D.ptr(s_d), D.ptr(v_d), D.ptr(o_d),
              n_elem, n_dof, D.ptr(off), D.ptr(ent), D.ptr(rows), 1, D.stream_ptr())
    out[...] = o_d.cpu().numpy()


def fused_atomic(edof, ke, scale, v, out) -> None:
    """red.global.add fused K v, accumulated into out."""
    _fused(edof, ke, scale, v, out, _lib.TF_SCATTER_ATOMIC)


def gather(edof, v):
    dt = np.asarray(v).dtype
    e_d = D.to_dev(edof, np.int32)
    v_d = D.to_dev(v, dt)
    u = D.torch().empty((edof.shape[0], 24), dtype=D.tdtype(dt), device=e_d.device)
    _lib.call(f"tf_gather_{_sfx(v)}", D.ptr(e_d), D.ptr(v_d), D.ptr(u), edof.shape[0],
              D.stream_ptr())
    return u.cpu().numpy()


def gemm(u_elem, ke, scale):
    dt = np.asarray(u_elem).dtype
    u_d = D.to_dev(u_elem, dt)
    f = D.torch().empty_like(u_d)
    ke_h = np.ascontiguousarray(ke, dtype=dt)
    s_d = D.to_dev(scale, dt)
    _lib.call(f"tf_gemm_{_sfx(u_elem)}", D.ptr(u_d), ke_h.ctypes.data, D.ptr(s_d),
              D.ptr(f), u_elem.shape[0], D.stream_ptr())
    return f.cpu().numpy()


def scatter_serial(edof, f_elem, acc) -> None:
    """acc += scatter(f_elem) in ascending element order, FP64 accumulation --
    bitwise _kernels_numba.py:129-132 (operator.py:107-114)."""
    dt = np.asarray(f_elem).dtype
    edof = np.ascontiguousarray(edof, dtype=np.int32)
    a_d = D.to_dev(acc, np.float64)
    e_d = D.to_dev(edof, np.int32)
    f_d = D.to_dev(f_elem, dt)
    off, ent = _csr(e_d, edof.shape[0], acc.shape[0])
    _lib.call(f"tf_scatter_pull_{_sfx(f_elem)}", D.ptr(off), D.ptr(ent), D.ptr(f_d), D.ptr(a_d), acc.shape[0],
              D.stream_ptr())
    acc[...] = a_d.cpu().numpy().astype(acc.dtype)


def scatter_atomic(edof, f_elem, acc) -> None:
    """acc += scatter(f_elem) with red.global.add (FP64), any order."""
    dt = np.asarray(f_elem).dtype
    a_d = D.to_dev(acc, np.float64)
    e_d = D.to_dev(edof, np.int32)
    f_d = D.to_dev(f_elem, dt)
    _lib.call(f"tf_scatter_{_sfx(f_elem)}", D.ptr(e_d), D.ptr(f_d), D.ptr(a_d), edof.shape[0],
              D.stream_ptr())
    acc[...] = a_d.cpu().numpy().astype(acc.dtype)




def _csr(e_d, n_elem, n_dof):
    """DOF -> (element*24 + row) entries in ascending element order (device)."""
    t = D.torch()
    off = t.empty(n_dof + 1, dtype=t.int64, device=e_d.device)
    ent = t.empty(n_elem * 24, dtype=t.int32, device=e_d.device)
    _lib.call("tf_edof_csr_build", D.ptr(e_d), n_elem, n_dof, D.ptr(off), D.ptr(ent), D.stream_ptr())
    return off, ent


def jacobi_diag(edof, ke_diag, scale, out) -> None:
    """out[edof[e, l]] += scale[e] * ke_diag[l] in ascending element order,
    FP64 accumulation -- bitwise _kernels_numba.py:217-226."""
    dt = np.asarray(scale).dtype
    edof = np.ascontiguousarray(edof, dtype=np.int32)
    a_d = D.to_dev(out, np.float64)
    kd = np.ascontiguousarray(ke_diag, dtype=dt)
    e_d = D.to_dev(edof, np.int32)
    s_d = D.to_dev(scale, dt)
    off, ent = _csr(e_d, edof.shape[0], out.shape[0])
    _lib.call(f"tf_jacobi_edof_pull_{_sfx(scale)}", D.ptr(off), D.ptr(ent), kd.ctypes.data, D.ptr(s_d),
              D.ptr(a_d), out.shape[0], D.stream_ptr())
    out[...] = a_d.cpu().numpy().astype(out.dtype)


def element_energies(edof, ke, u):
    u_d = D.to_dev(u, np.float64)
    out = D.torch().empty(edof.shape[0], dtype=D.torch().float64, device=u_d.device)
    ke_h = np.ascontiguousarray(ke, dtype=np.float64)
    e_d = D.to_dev(edof, np.int32)
    _lib.call("tf_energies_edof_f64", D.ptr(e_d), ke_h.ctypes.data,
              D.ptr(u_d), D.ptr(out), edof.shape[0], D.stream_ptr())
    return out.cpu().numpy()


# -- emulated bfloat16 contract (_kernels_numba.py:113-126, 166-211, 230-238) -----


def _fused_bf16(edof, ke, scale, v, out, mode):
    edof = np.ascontiguousarray(edof, dtype=np.int32)
    e_d = D.to_dev(edof, np.int32)
    s_d = D.to_dev(scale, np.float32)
    v_d = D.to_dev(v, np.float32)
    o_d = D.to_dev(out, np.float32)
    ke_h = np.ascontiguousarray(ke, dtype=np.float32)
    if mode == _lib.TF_SCATTER_COLORED:
        from .mesh import StructuredMesh
        from .operator import element_colouring

        n = edof.shape[0]
        order, offsets = element_colouring(StructuredMesh(n, 1, 1), edof)
        o_ = D.to_dev(order, np.int32)
        _lib.call("tf_matvec_edof_bf16", D.ptr(e_d), ke_h.ctypes.data, D.ptr(s_d), D.ptr(v_d), D.ptr(o_d),
                  n, mode, D.ptr(o_), offsets.ctypes.data, len(offsets) - 1, 0, D.stream_ptr())
    else:
        _lib.call("tf_matvec_edof_bf16", D.ptr(e_d), ke_h.ctypes.data, D.ptr(s_d), D.ptr(v_d), D.ptr(o_d),
                  edof.shape[0], mode, None, None, 0, 0, D.stream_ptr())
    out[...] = o_d.cpu().numpy()


def fused_serial_bf16(edof, ke, scale, v, out) -> None:
    """fused K v with per-term bf16(s K), v pre-quantized, out += (FP32) in the
    reference's element order -- bitwise _kernels_numba.py:166-177."""
    t = D.torch()
    edof = np.ascontiguousarray(edof, dtype=np.int32)
    n_elem, n_dof = edof.shape[0], out.shape[0]
    e_d = D.to_dev(edof, np.int32)
    s_d = D.to_dev(scale, np.float32)
    v_d = D.to_dev(v, np.float32)
    o_d = D.to_dev(out, np.float32)
    off, ent = _csr(e_d, n_elem, n_dof)
    rows = t.empty(n_elem * 24, dtype=t.float64, device=e_d.device)
    ke_h = np.ascontiguousarray(ke, dtype=np.float32)
    _lib.call("tf_matvec_edof_pull_bf16", D.ptr(e_d), ke_h.ctypes.data, D.ptr(s_d), D.ptr(v_d), D.ptr(o_d),
              n_elem, n_dof, D.ptr(off), D.ptr(ent), D.ptr(rows), 1, D.stream_ptr())
    out[...] = o_d.cpu().numpy()


def fused_atomic_bf16(edof, ke, scale, v, out) -> None:
    """red.global.add variant of fused_serial_bf16."""
    _fused_bf16(edof, ke, scale, v, out, _lib.TF_SCATTER_ATOMIC)


def gemm_bf16(u_elem, ke, scale):
    u_d = D.to_dev(u_elem, np.float32)
    f = D.torch().empty_like(u_d)
    ke_h = np.ascontiguousarray(ke, dtype=np.float32)
    s_d = D.to_dev(scale, np.float32)
    _lib.call("tf_gemm_bf16", D.ptr(u_d), ke_h.ctypes.data, D.ptr(s_d), D.ptr(f), u_elem.shape[0],
              D.stream_ptr())
    return f.cpu().numpy()


def jacobi_diag_bf16(edof, ke_diag, scale, out) -> None:
    """out[edof] += bf16(s_e ke_diag[l]) in FP32."""
    o_d = D.to_dev(out, np.float32)
    kd = np.ascontiguousarray(ke_diag, dtype=np.float32)
    e_d = D.to_dev(edof, np.int32)
    s_d = D.to_dev(scale, np.float32)
    _lib.call("tf_jacobi_edof_bf16", D.ptr(e_d), kd.ctypes.data, D.ptr(s_d), D.ptr(o_d), edof.shape[0],
              D.stream_ptr())
    out[...] = o_d.cpu().numpy()
