"""Matrix-free stiffness operator on B200 (mirrors reference operator.py:38-268).

``MatFreeOperator`` keeps the reference constructor and methods (apply,
__call__, diagonal, apply_fp64, element_energies, compliance, n_apply) and the
traffic/roofline helpers, but every evaluation runs in libtopofuse_b200.so on
the current CUDA device:

  * structured grids (edof == build_edof(mesh)): the index-free parity-block
    tile kernel (csrc/tf_tile.cu: element columns marching in z, no atomics,
    deterministic) with input masking and fixed-DOF pass-through fused in --
    ONE launch per apply (grid_kernel="pull": the dense node-centric kernel;
    exact=True: the reference's operation order, bitwise);
  * any other edof: the element-per-thread kernel with red.global.add
    (scatter="parallel_atomic") or the reference's serial order, bitwise
    (scatter="serial": row sums + ascending-element pull through a DOF CSR),
    constrained slots masked in the device edof copy;
  * variant="three_stage": gather -> batched element product -> FP64
    histogram scatter, intermediates genuinely materialised (operator.py:103-114).

Inputs may be numpy arrays (copied to/from the device, as a drop-in) or
torch CUDA tensors (stay resident; results are tensors).
"""

from __future__ import annotations

import hashlib
import os
import weakref
from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import _lib
from .element import SimpParams, simp_scale, unit_stiffness
from .mesh import BoundaryConditions, StructuredMesh, edof_is_structured
from .precision import FP64, Precision, get_precision

VARIANTS = ("three_stage", "fused")
SCATTER_MODES = ("serial", "parallel_atomic")
BACKENDS = ("b200",)

FLOPS_PER_ELEMENT = 2 * 24 * 24
INDEX_BYTES_PER_ELEMENT = 24 * 4
DENSITY_BYTES_PER_ELEMENT = 4

ENV_EXACT = "TOPOFUSE_B200_EXACT"  # 1 -> bitwise numba-order kernels for structured grids
# structured-grid kernels: parity-block element tiles (production), dense
# node-centric pull, and the bitwise reference-order pull
GRID_KERNELS = {"tile": 0, "exact": 1, "pull": 2, "edof": -1}  # "edof": force the general kernels


class DeviceProblem:
    """Device-resident connectivity/constraint data shared by every operator
    built on the same (mesh, edof, bcs) -- run_simp rebuilds the operator each
    iteration (simp.py:358-369) but this is uploaded once."""

    def __init__(self, mesh: StructuredMesh, edof: np.ndarray, bcs: BoundaryConditions):
        # no strong reference to the caller's edof or mesh: the cache entry
        # holding this object is keyed on edof and must die with it
        # (_device.IdCache), so keep a weakref and a private mesh copy
        self.mesh = StructuredMesh(mesh.nelx, mesh.nely, mesh.nelz)
        self.n_dof = mesh.n_dof
        self.n_elem = mesh.n_elem
        self.structured = edof_is_structured(mesh, edof)
        self.fixed_np = np.asarray(bcs.fixed_dofs, dtype=np.int64)
        self.fixed = D.to_dev(self.fixed_np, np.int64) if self.fixed_np.size else None
        self.grid = _lib.tf_grid(mesh.nelx, mesh.nely, mesh.nelz)
        # node bytes + per-(i,j)-column OR bytes, built on the device
        nbytes = mesh.n_nodes + 2 * (mesh.nelx + 1) * (mesh.nely + 1)
        t = D.torch()
        self.node_fixed = t.empty((nbytes + 3) // 4 * 4, dtype=t.uint8, device=D.require_cuda())
        _lib.call("tf_build_node_fixed", ctypes_ref(self.grid), D.ptr(self.fixed),
                  int(self.fixed_np.size), D.ptr(self.node_fixed), D.stream_ptr())
        self._edof_ref = weakref.ref(edof)
        self._edof_masked = None
        self._edof_raw = None
        self._colors = None
        self._csr = None
        self._merge = None
        self.pcg_handles = {}

    @property
    def _edof_np(self) -> np.ndarray:
        e = self._edof_ref()
        if e is None:  # pragma: no cover - the cache entry dies with edof
            raise _lib.TfError("device problem outlived its connectivity array")
        return e

    @property
    def edof_masked(self):
        if self._edof_masked is None:
            self._edof_masked = D.to_dev(D.masked_edof(self._edof_np, self.fixed_np, self.n_dof), np.int32)
        return self._edof_masked

    @property
    def edof_raw(self):
        if self._edof_raw is None:
            self._edof_raw = D.to_dev(np.ascontiguousarray(self._edof_np, dtype=np.int32), np.int32)
        return self._edof_raw

    def csr(self):
        """DOF -> (element, row) CSR in ascending element order (built once on
        the device, tf_edof_csr_build) and the FP64 row workspace of the
        bitwise fused_serial pull (tf_matvec_edof_pull_*)."""
        if self._csr is None:
            t = D.torch()
            n_rows = self.n_elem * 24
            off = t.empty(self.n_dof + 1, dtype=t.int64, device=self.edof_raw.device)
            ent = t.empty(n_rows, dtype=t.int32, device=off.device)
            _lib.call("tf_edof_csr_build", D.ptr(self.edof_raw), self.n_elem, self.n_dof, D.ptr(off), D.ptr(ent),
                      D.stream_ptr())
            rows = t.empty(n_rows, dtype=t.float64, device=off.device)
            self._csr = (off, ent, rows)
        return self._csr

    def merge_mask(self):
        """Per-element 16-bit mask of the (right corner of e, left corner of
        e+1) DOF pairs the atomic product sums in registers before one
        red.global (tf_edof_merge_mask, once per connectivity)."""
        if self._merge is None:
            t = D.torch()
            em = self.edof_masked
            self._merge = t.empty(self.n_elem, dtype=t.int16, device=em.device)
            _lib.call("tf_edof_merge_mask", D.ptr(em), self.n_elem, self.n_dof, D.ptr(self._merge), D.stream_ptr())
        return self._merge

    def colors(self):
        """Element colouring with no two same-colour elements sharing a DOF."""
        if self._colors is None:
            order, offsets = element_colouring(self.mesh, self._edof_np)
            self._colors = (D.to_dev(order, np.int32), np.ascontiguousarray(offsets, dtype=np.int64))
        return self._colors

    def __del__(self):
        for h in getattr(self, "pcg_handles", {}).values():
            try:
                _lib.load().tf_pcg_destroy(h)
            except Exception:  # pragma: no cover - interpreter teardown
                pass


def element_colouring(mesh: StructuredMesh, edof: np.ndarray):
    """Grid-parity colouring (8 colours) validated against edof; greedy otherwise."""
    e = np.arange(mesh.n_elem, dtype=np.int64)
    ex = e % mesh.nelx
    ey = (e // mesh.nelx) % mesh.nely
    ez = e // (mesh.nelx * mesh.nely)
    col = (ex & 1) | ((ey & 1) << 1) | ((ez & 1) << 2)
    ok = True
    for c in range(8):
        rows = edof[col == c]
        if rows.size and np.unique(rows).size != rows.size:
            ok = False
            break
    if not ok:
        if mesh.n_elem > 300_000:
            raise NotImplementedError("greedy colouring of large non-grid connectivity")
        col = np.zeros(mesh.n_elem, dtype=np.int64)
        used_by_dof = [set() for _ in range(int(edof.max()) + 1)]
        for i in range(mesh.n_elem):
            taken = set()
            for d in edof[i]:
                taken |= used_by_dof[d]
            c = 0
            while c in taken:
                c += 1
            col[i] = c
            for d in edof[i]:
                used_by_dof[d].add(c)
    order = np.argsort(col, kind="stable").astype(np.int32)
    counts = np.bincount(col, minlength=int(col.max()) + 1)
    offsets = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    return order, offsets


def _constraint_digest(bcs) -> bytes:
    """Content key of the constraint set (ids of dead objects are reused)."""
    f = np.ascontiguousarray(np.asarray(bcs.fixed_dofs, dtype=np.int64))
    return hashlib.sha1(f.tobytes()).digest()


def device_problem(mesh, edof, bcs) -> DeviceProblem:
    """Device data of (mesh, edof, bcs), cached on edof and keyed on the
    constraint CONTENT -- two load cases on one mesh with different supports
    never share constraint masks, whatever their object ids."""
    key = (mesh.nelx, mesh.nely, mesh.nelz, _constraint_digest(bcs))

    def make():
        return DeviceProblem(mesh, edof, bcs)

    return D.CACHE.get(edof, key, make)


def _sfx(dtype) -> str:
    return "f64" if np.dtype(dtype) == np.float64 else "f32"


class MatFreeOperator:
    """Matrix-free K(rho) (reference operator.py:38-162) evaluated on B200."""

    def __init__(
        self,
        mesh: StructuredMesh,
        edof: np.ndarray,
        bcs: BoundaryConditions,
        density: np.ndarray,
        simp: SimpParams = SimpParams(),
        precision: Precision | str = FP64,
        variant: str = "fused",
        scatter: str = "serial",
        nu: float = 0.3,
        backend: str | None = None,
        exact: bool | None = None,
        grid_kernel: str = "tile",
    ):
        if variant not in VARIANTS:
            raise ValueError(f"variant must be one of {VARIANTS}")
        if scatter not in SCATTER_MODES:
            raise ValueError(f"scatter must be one of {SCATTER_MODES}")
        if backend not in (None,) + BACKENDS:
            raise ValueError(f"unknown backend {backend!r}, expected b200")
        self.precision = get_precision(precision) if isinstance(precision, str) else precision
        # "bf16" is the reference's emulated-bfloat16 precision (FP32 storage,
        # per-term rounding): served by the general-edof bf16 kernels
        # (csrc/tf_bf16.cu) as the documented negative result, never by the
        # structured production kernels
        self.mesh = mesh
        self.edof = edof
        self.bcs = bcs
        self.simp = simp
        self.variant = variant
        self.scatter = scatter
        self.nu = nu
        self.backend_name = "b200"
        self.n_dof = mesh.n_dof
        self.fixed_dofs = bcs.fixed_dofs
        self.density = np.asarray(density, dtype=np.float64)
        if self.density.shape != (mesh.n_elem,):
            raise ValueError("density must have one entry per element")
        self.exact = bool(int(os.environ.get(ENV_EXACT, "0"))) if exact is None else bool(exact)
        if grid_kernel not in GRID_KERNELS:
            raise ValueError(f"grid_kernel must be one of {tuple(GRID_KERNELS)}")
        self.grid_kernel = "exact" if self.exact else grid_kernel

        self.ke64 = unit_stiffness(nu)
        self.scale64 = np.asarray(simp_scale(self.density, simp), dtype=np.float64)
        dt = self.precision.dtype
        self.ke = np.ascontiguousarray(self.ke64, dtype=dt)
        self.scale = self.scale64.astype(dt)
        self.n_apply = 0

        self.dev = device_problem(mesh, edof, bcs)
        self._scale_dev = D.to_dev(self.scale, dt)
        self._scale64_dev = None

    # -- masks -------------------------------------------------------------------
    @property
    def free_mask(self) -> np.ndarray:
        return self.bcs.free_mask(self.n_dof)

    @property
    def structured(self) -> bool:
        """True when the index-free structured kernels serve this operator."""
        return self.dev.structured and self.grid_kernel != "edof" and not self.precision.quantized

    @property
    def grid_variant(self) -> int:
        return GRID_KERNELS[self.grid_kernel]

    # -- device-level entry points (torch tensors in, torch tensors out) ----------
    def apply_device(self, x, out=None, ke=None, scale=None, dtype=None):
        """w = K x on device (masked input, fixed pass-through), one launch on a grid."""
        t = D.torch()
        dt = np.dtype(dtype or self.precision.dtype)
        ke = self.ke if ke is None else ke
        scale = self._scale_dev if scale is None else scale
        if out is None:
            out = t.empty(self.n_dof, dtype=D.tdtype(dt), device=x.device)
        sfx = _sfx(dt)
        st = D.stream_ptr()
        dev = self.dev
        if self.precision.quantized:
            return self._apply_bf16(x, out, ke, scale, np.dtype(dt) == np.float64)
        if self.variant == "fused" and self.structured:
            _lib.call(f"tf_matvec_grid_{sfx}", ctypes_ref(dev.grid), ke.ctypes.data, D.ptr(scale),
                      D.ptr(x), D.ptr(out), D.ptr(dev.node_fixed),
                      _lib.TF_MASK_INPUT | _lib.TF_PASS_FIXED, self.grid_variant, st)
            return out
        if self.variant == "fused":
            out.zero_()
            if self.scatter == "parallel_atomic" and os.environ.get("TF_EDOF_MERGED", "1") == "1":
                _lib.call(f"tf_matvec_edof_merged_{sfx}", D.ptr(dev.edof_masked), D.ptr(dev.merge_mask()),
                          ke.ctypes.data, D.ptr(scale), D.ptr(x), D.ptr(out), self.mesh.n_elem, st)
            elif self.scatter == "parallel_atomic":  # TF_EDOF_MERGED=0: the v2 kernel (A/B)
                _lib.call(f"tf_matvec_edof_{sfx}", D.ptr(dev.edof_masked), ke.ctypes.data,
                          D.ptr(scale), D.ptr(x), D.ptr(out), self.mesh.n_elem,
                          _lib.TF_SCATTER_ATOMIC, None, None, 0, st)
            elif os.environ.get("TF_EDOF_COLORED") == "1":  # colour-ordered passes (A/B)
                order, offsets = dev.colors()
                _lib.call(f"tf_matvec_edof_{sfx}", D.ptr(dev.edof_masked), ke.ctypes.data,
                          D.ptr(scale), D.ptr(x), D.ptr(out), self.mesh.n_elem,
                          _lib.TF_SCATTER_COLORED, D.ptr(order), offsets.ctypes.data,
                          len(offsets) - 1, st)
            else:  # serial: the reference's element order, bitwise (tf_edof_pull.cu)
                off, ent, rows = dev.csr()
                _lib.call(f"tf_matvec_edof_pull_{sfx}", D.ptr(dev.edof_masked), ke.ctypes.data,
                          D.ptr(scale), D.ptr(x), D.ptr(out), self.mesh.n_elem, self.n_dof,
                          D.ptr(off), D.ptr(ent), D.ptr(rows), 0, st)
        else:
            n = self.mesh.n_elem
            u_elem = t.empty((n, 24), dtype=D.tdtype(dt), device=x.device)
            f_elem = t.empty_like(u_elem)
            acc = t.zeros(self.n_dof, dtype=t.float64, device=x.device)
            em = dev.edof_masked
            _lib.call(f"tf_gather_{sfx}", D.ptr(em), D.ptr(x), D.ptr(u_elem), n, st)
            _lib.call(f"tf_gemm_{sfx}", D.ptr(u_elem), ke.ctypes.data, D.ptr(scale), D.ptr(f_elem), n, st)
            _lib.call(f"tf_scatter_{sfx}", D.ptr(em), D.ptr(f_elem), D.ptr(acc), n, st)
            out.copy_(acc)
        if dev.fixed is not None:
            _lib.call(f"tf_pass_fixed_{sfx}", D.ptr(dev.fixed), int(dev.fixed_np.size), D.ptr(x),
                      D.ptr(out), st)
        return out

    def _apply_bf16(self, x, out, ke, scale, fp64):
        """Emulated-bf16 apply (operator.py:83-117) or its FP64 evaluation
        (apply_fp64, operator.py:143-152): quantized input and per-term
        bf16(s_e K_ij), pass-through of the raw input on fixed DOFs."""
        t = D.torch()
        dev = self.dev
        st = D.stream_ptr()
        ke32 = np.ascontiguousarray(self.ke, dtype=np.float32)
        s32 = self._scale_dev
        n = self.mesh.n_elem
        if fp64:
            out.zero_()
            _lib.call("tf_matvec_edof_bf16_f64", D.ptr(dev.edof_masked), ke32.ctypes.data, D.ptr(s32),
                      D.ptr(x), D.ptr(out), n, st)
            sfx = "f64"
        elif self.variant == "fused":
            out.zero_()
            if self.scatter == "parallel_atomic":
                _lib.call("tf_matvec_edof_bf16", D.ptr(dev.edof_masked), ke32.ctypes.data, D.ptr(s32),
                          D.ptr(x), D.ptr(out), n, _lib.TF_SCATTER_ATOMIC, None, None, 0, 1, st)
            else:
                order, offsets = dev.colors()
                _lib.call("tf_matvec_edof_bf16", D.ptr(dev.edof_masked), ke32.ctypes.data, D.ptr(s32),
                          D.ptr(x), D.ptr(out), n, _lib.TF_SCATTER_COLORED, D.ptr(order),
                          offsets.ctypes.data, len(offsets) - 1, 1, st)
            sfx = "f32"
        else:
            xq = t.empty_like(x)
            _lib.call("tf_round_bf16", self.n_dof, D.ptr(x), D.ptr(xq), st)
            u_elem = t.empty((n, 24), dtype=t.float32, device=x.device)
            f_elem = t.empty_like(u_elem)
            acc = t.zeros(self.n_dof, dtype=t.float64, device=x.device)
            em = dev.edof_masked
            _lib.call("tf_gather_f32", D.ptr(em), D.ptr(xq), D.ptr(u_elem), n, st)
            _lib.call("tf_gemm_bf16", D.ptr(u_elem), ke32.ctypes.data, D.ptr(s32), D.ptr(f_elem), n, st)
            _lib.call("tf_scatter_f32", D.ptr(em), D.ptr(f_elem), D.ptr(acc), n, st)
            out.copy_(acc)
            sfx = "f32"
        if dev.fixed is not None:
            _lib.call(f"tf_pass_fixed_{sfx}", D.ptr(dev.fixed), int(dev.fixed_np.size), D.ptr(x),
                      D.ptr(out), st)
        return out

    def diagonal_device(self):
        """(diag, inv_diag) device tensors in the working dtype."""
        t = D.torch()
        dt = self.precision.dtype
        sfx = _sfx(dt)
        dev = self.dev
        kd = np.ascontiguousarray(np.diag(self.ke), dtype=dt)
        diag = t.empty(self.n_dof, dtype=D.tdtype(dt), device=self._scale_dev.device)
        inv = t.empty_like(diag)
        if self.precision.quantized:  # jacobi_diag_bf16 (operator.py:122-126), FP32 accumulation
            diag.zero_()
            _lib.call("tf_jacobi_edof_bf16", D.ptr(dev.edof_raw), kd.ctypes.data, D.ptr(self._scale_dev),
                      D.ptr(diag), self.mesh.n_elem, D.stream_ptr())
            if dev.fixed is not None:
                diag[dev.fixed] = 1.0
            return diag, 1.0 / diag
        if self.structured:
            _lib.call(f"tf_jacobi_grid_{sfx}", ctypes_ref(dev.grid), kd.ctypes.data,
                      D.ptr(self._scale_dev), D.ptr(diag), D.ptr(inv), D.ptr(dev.node_fixed),
                      D.stream_ptr())
        else:
            # the reference's jacobi_diag order (ascending element per DOF): bitwise
            acc = t.zeros(self.n_dof, dtype=t.float64, device=diag.device)
            off, ent, _ = dev.csr()
            _lib.call(f"tf_jacobi_edof_pull_{sfx}", D.ptr(off), D.ptr(ent), kd.ctypes.data,
                      D.ptr(self._scale_dev), D.ptr(acc), self.n_dof, D.stream_ptr())
            diag.copy_(acc)
            if dev.fixed is not None:
                diag[dev.fixed] = 1.0
            inv = 1.0 / diag
        return diag, inv

    def energies_device(self, u64):
        t = D.torch()
        out = t.empty(self.mesh.n_elem, dtype=t.float64, device=u64.device)
        ke = np.ascontiguousarray(self.ke64, dtype=np.float64)
        if self.structured:
            _lib.call("tf_energies_grid_f64", ctypes_ref(self.dev.grid), ke.ctypes.data,
                      D.ptr(u64), D.ptr(out), D.stream_ptr())
        else:
            _lib.call("tf_energies_edof_f64", D.ptr(self.dev.edof_raw), ke.ctypes.data,
                      D.ptr(u64), D.ptr(out), self.mesh.n_elem, D.stream_ptr())
        return out

    def apply_stream(self, host_in, host_out):
        """w_i = K v_i for a sequence of HOST vectors, copies overlapped.

        `host_in` / `host_out`: equal-length sequences of pinned torch CPU
        tensors (n_dof, working dtype).  Three CUDA streams pipeline the
        H2D copy of v_{i+1}, the kernel on v_i and the D2H copy of w_{i-1}
        through double-buffered device vectors, so PCIe traffic in both
        directions overlaps the matvecs.  Returns after all copies land.
        """
        t = D.torch()
        dev = self._scale_dev.device
        tdt = D.tdtype(self.precision.dtype)
        if self.variant == "fused" and self.structured and self.grid_kernel == "tile" and host_in:
            # native pipeline (csrc/tf_stream.cu): the whole schedule enqueued from C
            import ctypes

            n = len(host_in)
            buf = getattr(self, "_native_stream_bufs", None)
            if buf is None or buf[0].dtype != tdt:
                buf = (t.empty(2 * self.n_dof, dtype=tdt, device=dev), t.empty(2 * self.n_dof, dtype=tdt, device=dev))
                self._native_stream_bufs = buf
            ins = (ctypes.c_void_p * n)(*[h.data_ptr() for h in host_in])
            outs = (ctypes.c_void_p * n)(*[h.data_ptr() for h in host_out])
            sfx = _sfx(self.precision.dtype)
            rc = getattr(_lib.load(), f"tf_matvec_grid_stream_{sfx}")(
                ctypes_ref(self.dev.grid), self.ke.ctypes.data, D.ptr(self._scale_dev),
                D.ptr(self.dev.node_fixed), _lib.TF_MASK_INPUT | _lib.TF_PASS_FIXED, n, ins, outs,
                D.ptr(buf[0]), D.ptr(buf[1]), D.stream_ptr())
            if rc == _lib.TF_OK:
                self.n_apply += n
                return host_out
            if rc != _lib.TF_ERR_UNSUPPORTED:  # a Ke without the parity structure takes the path below
                _lib.check(rc, "tf_matvec_grid_stream")
        cur = t.cuda.current_stream()
        if getattr(self, "_stream_ctx", None) is None:  # streams/buffers reused across calls
            self._stream_ctx = (
                (t.cuda.Stream(), t.cuda.Stream(), t.cuda.Stream()),
                [t.empty(self.n_dof, dtype=tdt, device=dev) for _ in range(2)],
                [t.empty(self.n_dof, dtype=tdt, device=dev) for _ in range(2)],
                [[t.cuda.Event() for _ in range(2)] for _ in range(3)],
            )
        (s_in, s_k, s_out), xin, wout, (h2d_done, k_done, d2h_done) = self._stream_ctx
        for s_ in (s_in, s_k, s_out):
            s_.wait_stream(cur)
        for i, (hv, hw) in enumerate(zip(host_in, host_out)):
            b = i & 1
            with t.cuda.stream(s_in):
                if i >= 2:
                    s_in.wait_event(k_done[b])      # xin[b] consumed by kernel i-2
                xin[b].copy_(hv, non_blocking=True)
                h2d_done[b].record(s_in)
            with t.cuda.stream(s_k):
                s_k.wait_event(h2d_done[b])
                if i >= 2:
                    s_k.wait_event(d2h_done[b])     # wout[b] drained by copy i-2
                self.apply_device(xin[b], out=wout[b])
                k_done[b].record(s_k)
            with t.cuda.stream(s_out):
                s_out.wait_event(k_done[b])
                hw.copy_(wout[b], non_blocking=True)
                d2h_done[b].record(s_out)
            self.n_apply += 1
        for s_ in (s_in, s_k, s_out):
            cur.wait_stream(s_)
        return host_out

    # -- reference API -------------------------------------------------------------
    def apply(self, v):
        """w = K v (operator.py:90-117)."""
        dt = self.precision.dtype
        if D.is_tensor(v) and v.is_cuda:
            x = v.to(D.tdtype(dt)).contiguous()
            out = self.apply_device(x)
            self.n_apply += 1
            return out
        x = D.to_dev(np.asarray(v), dt)
        out = self.apply_device(x)
        self.n_apply += 1
        return out.cpu().numpy()

    def __call__(self, v):
        return self.apply(v)

    def diagonal(self) -> np.ndarray:
        """Jacobi diagonal, 1.0 on fixed DOFs (operator.py:122-132)."""
        d, _ = self.diagonal_device()
        return d.cpu().numpy()

    def apply_fp64(self, v):
        """Exact FP64 matvec of the master data (operator.py:134-155)."""
        if self._scale64_dev is None:
            self._scale64_dev = D.to_dev(self.scale64, np.float64)
        tensor_in = D.is_tensor(v) and v.is_cuda
        x = v.to(D.torch().float64).contiguous() if tensor_in else D.to_dev(np.asarray(v), np.float64)
        if self.precision.quantized:  # the quantized system the solver saw, FP64 accumulation
            out = self._apply_bf16(x, D.torch().empty_like(x), None, None, True)
            return out if tensor_in else out.cpu().numpy()
        out = self.apply_device(x, ke=np.ascontiguousarray(self.ke64), scale=self._scale64_dev,
                                dtype=np.float64)
        return out if tensor_in else out.cpu().numpy()

    def element_energies(self, u):
        """u_e^T Ke u_e per element, FP64 (operator.py:157-159)."""
        tensor_in = D.is_tensor(u) and u.is_cuda
        u64 = u.to(D.torch().float64).contiguous() if tensor_in else D.to_dev(np.asarray(u), np.float64)
        out = self.energies_device(u64)
        return out if tensor_in else out.cpu().numpy()

    def compliance(self, f, u) -> float:
        if D.is_tensor(u):
            u = u.double().cpu().numpy()
        return float(np.dot(np.asarray(f, np.float64), np.asarray(u, np.float64)))


def ctypes_ref(struct):
    import ctypes

    return ctypes.addressof(struct)


def jacobi_diagonal(op: MatFreeOperator) -> np.ndarray:
    return op.diagonal()


# -- traffic model and roofline (reference operator.py:172-268) ---------------------


@dataclass(frozen=True)
class TrafficReport:
    variant: str
    precision: str
    scalar_bytes: int
    bytes_element_data: int
    bytes_with_indices: int
    flops_per_element: int
    intensity_ideal: float
    intensity_profile: float


def traffic_model(variant: str, precision: Precision | str) -> TrafficReport:
    """The paper's per-element byte model; element data is
    touched twice by the fused kernel and four times by three-stage."""
    if variant not in VARIANTS:
        raise ValueError(f"variant must be one of {VARIANTS}")
    prec = get_precision(precision) if isinstance(precision, str) else precision
    w = prec.scalar_bytes
    element_data = (4 if variant == "three_stage" else 2) * 24 * w
    with_idx = element_data + INDEX_BYTES_PER_ELEMENT + DENSITY_BYTES_PER_ELEMENT
    return TrafficReport(variant, prec.tag, w, element_data, with_idx, FLOPS_PER_ELEMENT,
                         FLOPS_PER_ELEMENT / element_data, FLOPS_PER_ELEMENT / with_idx)


@dataclass(frozen=True)
class RooflineConfig:
    peak_flops: float
    bandwidth: float

    def __post_init__(self):
        if self.peak_flops <= 0 or self.bandwidth <= 0:
            raise ValueError("roofline ceilings must be positive")

    @property
    def ridge(self) -> float:
        return self.peak_flops / self.bandwidth


# The reference's study device (RTX 4090 datasheet, operator.py:232-236) ...
DEVICE_CEILINGS = {
    "fp64": RooflineConfig(peak_flops=1.29e12, bandwidth=1.008e12),
    "fp32": RooflineConfig(peak_flops=82.6e12, bandwidth=1.008e12),
    "bf16": RooflineConfig(peak_flops=165.2e12, bandwidth=1.008e12),
}


def roofline_bound(config: RooflineConfig, intensity: float) -> float:
    if intensity <= 0:
        raise ValueError("arithmetic intensity must be positive")
    return min(config.peak_flops, intensity * config.bandwidth)


def effective_bandwidth(bytes_per_element: int, n_elem: int, seconds: float) -> float:
    if seconds <= 0:
        raise ValueError("wall time must be positive")
    return bytes_per_element * n_elem / seconds


def memory_footprint(n_elem: int, n_dof: int, variant: str, precision: Precision | str) -> int:
    prec = get_precision(precision) if isinstance(precision, str) else precision
    w = prec.scalar_bytes
    total = n_elem * INDEX_BYTES_PER_ELEMENT + n_elem * (8 + w) + 576 * w + 3 * n_dof * w
    if variant == "three_stage":
        total += 2 * n_elem * 24 * w
    return total


def compulsory_bytes(n_elem: int, n_dof: int, precision: str, structured: bool) -> int:
    """Algorithmic DRAM bytes of one fused matvec.

    General edof contract: edof row (96 B) + scale + v read once + w written
    once.  Structured (index-free) kernel: scale + v + w + the node mask byte.
    """
    w = 8 if precision == "fp64" else 4
    if structured:
        return n_elem * w + 2 * n_dof * w + n_dof // 3
    return n_elem * (96 + w) + 2 * n_dof * w
