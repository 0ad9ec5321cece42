"""Jacobi-PCG on B200 (mirrors reference solver.py:22-190).

``pcg(apply_op, b, diag, config, x0)`` keeps the reference signature.  When
``apply_op`` is a ``MatFreeOperator`` (or its bound ``apply``) the whole
solve runs on the device as one CUDA-graph launch (tf_pcg_solve: conditional
while loop, fused matvec+dot, deterministic reductions, FP32 scalar rounding
mirroring numpy).  Any other callable gets the same recurrence with the
vectors held as CUDA tensors and the callable evaluated on host arrays.
"""

from __future__ import annotations

import ctypes
import math
import os
import time
from dataclasses import dataclass, replace

import numpy as np

from . import _device as D
from . import _lib
from .operator import MatFreeOperator


class DivergenceError(RuntimeError):
    """Non-finite CG recurrence values (solver.py:22-27)."""

    def __init__(self, iteration: int, detail: str):
        super().__init__(f"CG diverged at iteration {iteration}: {detail}")
        self.iteration = iteration


@dataclass(frozen=True)
class CgConfig:
    rel_tol: float = 1e-5
    max_iter: int = 1000
    recompute_every: int = 50
    quantize_krylov: bool = False

    def __post_init__(self):
        if self.rel_tol <= 0 or self.max_iter < 1 or self.recompute_every < 0:
            raise ValueError("invalid CG configuration")


@dataclass
class SolveReport:
    converged: bool
    termination: str
    iterations: int
    rel_residual: float
    residual_history: np.ndarray
    matvecs: int
    wall_time: float
    compliance: float | None = None
    precision: str = ""
    variant: str = ""
    verified_rel_residual: float | None = None


def _operator_of(apply_op):
    if isinstance(apply_op, MatFreeOperator):
        return apply_op
    owner = getattr(apply_op, "__self__", None)
    if isinstance(owner, MatFreeOperator) and getattr(apply_op, "__name__", "") in ("apply", "__call__"):
        return owner
    return None


def pcg(apply_op, b, diag, config: CgConfig = CgConfig(), x0=None):
    """Preconditioned CG in b's storage precision (solver.py:57-147)."""
    op = _operator_of(apply_op)
    if config.quantize_krylov and (op is None or op.precision.tag == "fp64"):
        raise ValueError("quantize_krylov needs a fp32/bf16 MatFreeOperator (FP32 storage)")
    if op is not None:
        return device_pcg(op, b, diag, config, x0)
    return _generic_pcg(apply_op, b, diag, config, x0)


# environment overrides read when a handle is planned (tf_pcg_create)
_PLAN_ENV = ("TF_PCG_RESIDENT", "TF_PCG_FUSED", "TF_PCG_ONEX", "TF_PCG_RES_BY", "TF_PCG_RES_OZ",
             "TF_PCG_RES_LEAN", "TF_RES_ISO32")


def _pcg_handle(op: MatFreeOperator, graph_only: bool = False):
    """One device PCG per (device problem, precision, kernel variant); graph_only
    forces the plain 3-kernel graph protocol (quantize_krylov rounds p and r
    in its direction kernel)."""
    dev = op.dev
    # the protocol overrides and the element matrix (copied into the handle
    # once, by tf_pcg_create) are fixed at handle creation: part of the key
    key = (op.precision.tag, np.ascontiguousarray(op.ke).tobytes(), op.grid_variant,
           op.variant == "fused" and op.structured,
           graph_only) + tuple(os.environ.get(v) for v in _PLAN_ENV)
    h = dev.pcg_handles.get(key)
    if h is not None:
        return h
    desc = _lib.tf_pcg_desc()
    desc.precision = {"fp64": 64, "fp32": 32, "bf16": 16}[op.precision.tag]
    desc.structured = 1 if (op.structured and op.variant == "fused") else 0
    desc.grid = dev.grid
    desc.edof = 0 if desc.structured else D.ptr(dev.edof_masked)
    desc.n_elem = op.mesh.n_elem
    desc.n_dof = op.n_dof
    op._ke_keepalive = np.ascontiguousarray(op.ke)
    desc.ke = op._ke_keepalive.ctypes.data
    desc.node_fixed = D.ptr(dev.node_fixed)
    desc.fixed = D.ptr(dev.fixed)
    desc.n_fixed = int(dev.fixed_np.size)
    desc.grid_variant = max(op.grid_variant, 0)
    desc.flags = 1 if graph_only else 0
    out = ctypes.c_void_p()
    _lib.call("tf_pcg_create", ctypes.byref(out), ctypes.byref(desc), D.stream_ptr())
    dev.pcg_handles[key] = out
    return out


PCG_PROTOCOLS = ("graph", "fused_graph", "resident")


def pcg_protocol(op: MatFreeOperator) -> str:
    """Device protocol of op's PCG handle (include/topofuse_b200.h tf_pcg_protocol):
    "resident" = the whole solve in one cooperative kernel with the owned CG
    vectors in shared memory; "fused_graph"/"graph" = one CUDA graph of 2/3
    kernels per iteration."""
    return PCG_PROTOCOLS[_lib.load().tf_pcg_protocol(_pcg_handle(op))]


def device_pcg(op: MatFreeOperator, b, diag, config: CgConfig = CgConfig(), x0=None,
               return_device: bool = False):
    """Device-resident solve; numpy in -> numpy out unless return_device."""
    t = D.torch()
    t0 = time.perf_counter()
    dt = np.asarray(b).dtype if not D.is_tensor(b) else np.dtype(str(b.dtype).replace("torch.", ""))
    if np.dtype(dt) != np.dtype(op.precision.dtype):
        raise ValueError(f"rhs dtype {dt} does not match operator precision {op.precision.tag}")
    b_d = D.to_dev(b, dt)
    if D.is_tensor(diag) and diag.is_cuda:
        inv_d = 1.0 / diag.to(D.tdtype(dt))
    else:
        # inv_diag = 1 / diag in the storage dtype (solver.py:95)
        inv_d = D.to_dev(1.0 / np.asarray(diag, dtype=dt), dt)
    x_d = t.empty_like(b_d)
    has_x0 = x0 is not None
    if has_x0:
        x_d.copy_(D.to_dev(x0, dt))
    hist = t.zeros(config.max_iter + 1, dtype=t.float64, device=b_d.device)
    h = _pcg_handle(op, graph_only=bool(config.quantize_krylov))
    _lib.call("tf_pcg_set_quantize_krylov", h, 1 if config.quantize_krylov else 0)
    rep = _lib.tf_pcg_report()
    _lib.call("tf_pcg_solve", h, D.ptr(op._scale_dev), D.ptr(b_d), D.ptr(inv_d), D.ptr(x_d),
              1 if has_x0 else 0, float(config.rel_tol), int(config.max_iter),
              int(config.recompute_every), D.ptr(hist), ctypes.byref(rep))
    term = _lib.TERMINATIONS[rep.termination]
    if term == "diverged":
        raise DivergenceError(rep.iterations, "non-finite curvature or residual")
    n_hist = rep.iterations + 1
    history = hist[:n_hist].cpu().numpy()
    if term == "breakdown":
        history = history[: rep.iterations]
    op.n_apply += rep.matvecs
    report = SolveReport(
        converged=(term == "converged"),
        termination=term,
        iterations=int(rep.iterations),
        rel_residual=float(rep.rel_residual),
        residual_history=np.asarray(history),
        matvecs=int(rep.matvecs),
        wall_time=time.perf_counter() - t0,
    )
    if return_device:
        return x_d, report
    return x_d.cpu().numpy(), report


def _generic_pcg(apply_op, b, diag, config: CgConfig, x0):
    """Same recurrence for an arbitrary callable; vectors live on the GPU."""
    t = D.torch()
    dev = D.require_cuda()
    t0 = time.perf_counter()
    b_np = np.ascontiguousarray(b)
    dt = b_np.dtype
    tdt = D.tdtype(dt)

    def A(vec):
        return t.from_numpy(np.ascontiguousarray(apply_op(vec.cpu().numpy()), dtype=dt)).to(dev)

    def dot(a, c):
        return float(np.asarray(t.dot(a, c).cpu().numpy(), dtype=dt))

    def norm(a):
        return float(np.asarray(t.linalg.vector_norm(a).cpu().numpy(), dtype=dt))

    bb = t.from_numpy(b_np).to(dev)
    bnorm = norm(bb)
    if bnorm == 0.0:
        return np.zeros_like(b_np), SolveReport(True, "converged", 0, 0.0, np.zeros(1), 0,
                                                time.perf_counter() - t0)
    mv = 0
    if x0 is None:
        x = t.zeros_like(bb)
        r = bb.clone()
    else:
        x = t.from_numpy(np.array(x0, dtype=dt)).to(dev)
        r = bb - A(x)
        mv += 1
    inv = t.from_numpy(np.ascontiguousarray(1.0 / np.asarray(diag, dtype=dt))).to(dev)
    z = r * inv
    p = z.clone()
    rz = dot(r, z)
    rel = norm(r) / bnorm
    hist = [rel]
    term = "converged" if rel <= config.rel_tol else "max_iter"
    done = rel <= config.rel_tol
    it = 0
    while not done and it < config.max_iter:
        it += 1
        q = A(p)
        mv += 1
        pq = dot(p, q)
        if not (math.isfinite(pq) and math.isfinite(rz)):
            raise DivergenceError(it, "non-finite curvature or residual product")
        if pq <= 0.0:
            term = "breakdown"
            break
        alpha = t.tensor(rz / pq, dtype=tdt, device=dev)
        x = x + alpha * p
        if config.recompute_every and it % config.recompute_every == 0:
            r = bb - A(x)
            mv += 1
        else:
            r = r - alpha * q
        rn = norm(r)
        if not math.isfinite(rn):
            raise DivergenceError(it, "non-finite residual norm")
        rel = rn / bnorm
        hist.append(rel)
        if rel <= config.rel_tol:
            term, done = "converged", True
            break
        z = r * inv
        rz_new = dot(r, z)
        beta = t.tensor(rz_new / rz, dtype=tdt, device=dev)
        p = z + beta * p
        rz = rz_new
    return x.cpu().numpy(), SolveReport(term == "converged", term, it, rel, np.asarray(hist), mv,
                                        time.perf_counter() - t0)


def solve_equilibrium(op: MatFreeOperator, f, config: CgConfig = CgConfig(), x0=None):
    """K(rho) u = f with the verified-residual floor rule (solver.py:150-183)."""
    rhs = np.ascontiguousarray(f, dtype=op.precision.dtype)
    diag_d, _ = op.diagonal_device()
    if op.precision.quantized and config.recompute_every:
        # a residual recomputed through the rounding operator sits O(eps kappa)
        # from the recurrence: quantized solves skip the refresh (solver.py:171-172)
        config = replace(config, recompute_every=0)
    u, report = pcg(op.apply, rhs, diag_d, config, x0=x0)
    report.compliance = op.compliance(f, u)
    report.precision = op.precision.tag
    report.variant = op.variant
    fnorm = float(np.linalg.norm(np.asarray(f, dtype=np.float64)))
    verified = 0.0 if fnorm == 0.0 else fp64_relative_residual(op, f, u)
    report.verified_rel_residual = verified
    if report.converged and verified > 2.0 * config.rel_tol:
        report.converged = False
        report.termination = "floor"
    return u, report


def fp64_relative_residual(op: MatFreeOperator, f, u) -> float:
    """||f - K u|| / ||f|| through the FP64 device matvec (solver.py:186-190)."""
    f64 = np.asarray(f, dtype=np.float64)
    r = f64 - op.apply_fp64(np.asarray(u, dtype=np.float64))
    return float(np.linalg.norm(r) / np.linalg.norm(f64))


@dataclass(frozen=True)
class IrConfig:
    inner_tol: float = 1e-3
    outer_tol: float = 1e-5
    max_outer: int = 8
    stagnation_drop: float = 0.05


@dataclass
class IrReport:
    converged: bool
    stagnated: bool
    outer_steps: int
    inner_iterations: list
    total_inner: int
    outer_residuals: list
    compliance: float
    wall_time: float


def solve_refined(op_outer: MatFreeOperator, op_inner: MatFreeOperator, f, ir: IrConfig = IrConfig(),
                  cg: CgConfig = CgConfig()):
    """Iterative refinement (solver.py:211-262): FP32 outer residuals through
    op_outer, inner corrections solved with op_inner (BF16) to ir.inner_tol
    with the refresh disabled; stops on the outer tolerance, the outer cap, or
    two consecutive outer reductions below ir.stagnation_drop (the eps*kappa
    barrier).  Vectors stay on the device; this reproduces the paper's
    negative result, it is not a production solver."""
    t = D.torch()
    t0 = time.perf_counter()
    dt = op_outer.precision.dtype
    rhs = D.to_dev(np.ascontiguousarray(f, dtype=dt), dt)
    fnorm = float(t.linalg.vector_norm(rhs).cpu())
    u = t.zeros_like(rhs)
    r = rhs.clone()
    diag_inner, _ = op_inner.diagonal_device()
    inner_cfg = CgConfig(rel_tol=ir.inner_tol, max_iter=cg.max_iter, recompute_every=0,
                         quantize_krylov=cg.quantize_krylov)
    outer = [1.0]
    inner_its = []
    converged = stagnated = False
    for _ in range(ir.max_outer):
        e, rep = device_pcg(op_inner, r.to(D.tdtype(op_inner.precision.dtype)), diag_inner, inner_cfg,
                            return_device=True)
        inner_its.append(rep.iterations)
        u = u + e.to(u.dtype)
        r = rhs - op_outer.apply(u)
        rel = float(t.linalg.vector_norm(r).cpu()) / fnorm
        outer.append(rel)
        if rel <= ir.outer_tol:
            converged = True
            break
        if len(outer) >= 3:
            drops = [1.0 - outer[-1] / outer[-2], 1.0 - outer[-2] / outer[-3]]
            if all(d < ir.stagnation_drop for d in drops):
                stagnated = True
                break
    u_np = u.cpu().numpy()
    return u_np, IrReport(converged, stagnated, len(inner_its), inner_its, int(sum(inner_its)), outer,
                          op_outer.compliance(f, u_np), time.perf_counter() - t0)


__all__ = ["CgConfig", "DivergenceError", "IrConfig", "IrReport", "SolveReport", "device_pcg",
           "fp64_relative_residual", "pcg", "solve_equilibrium", "solve_refined", "replace"]
