"""Device-resident SIMP iteration (reference simp.py:324-448 on B200).

Every per-element field lives on the GPU for the whole run: density filter
(structured stencil) and Heaviside projection, SIMP scale, Jacobi diagonal,
the PCG solve (one graph launch), compliance/grayness reductions, element
energies, the sensitivity chain (filter transpose) and the OC bisection (one
cooperative kernel).  The host only sees scalars (compliance, grayness, CG
report, volume) -- exactly what the selection/restart rules consume -- and
copies the selected/final fields out once at the end.

Used by ``simp.run_simp`` on structured grids with filter reach <= 3, for
both volume constraints (``volume_on="raw"``, the reference default: one
cooperative OC kernel; ``"projected"``: device filter/projection per
multiplier under the host bisection walk).
"""

from __future__ import annotations

import ctypes
import time

import numpy as np

from . import _device as D
from . import _lib
from .element import RHO_MIN, SimpParams
from .mesh import build_edof
from .operator import MatFreeOperator, ctypes_ref
from .precision import get_precision
from .solver import device_pcg


class _Selected:
    def __init__(self, it, c, g, rho, rho_phys, u, p, beta):
        self.iteration, self.compliance, self.grayness = it, c, g
        self.rho, self.rho_phys, self.u = rho, rho_phys, u
        self.p, self.beta = p, beta


def _oc_projected(n, grid, rmin, inv_rs, rho, dc, dh, s, vf, rho_new, work, stats, st):
    """oc_update on the projected volume (reference simp.py:393-401), device
    resident: dv = max(F^T dh, 1e-12); every multiplier's volume is
    mean(H_beta(F cand)) evaluated by the stencil filter, projection and a
    fixed-order reduction; the bracket/bisection walk is oc_bisect
    (slab_simp.py), validated step for step against oc_update."""
    t = D.torch()
    from .slab_simp import oc_bisect

    dv = t.empty_like(rho)
    _lib.call("tf_filter_grid_f64", ctypes_ref(grid), float(rmin), D.ptr(inv_rs), D.ptr(dh), D.ptr(dv), 1, st)
    dv.clamp_(min=1e-12)
    if float(dc.max()) > 1e-12:
        raise ValueError("compliance sensitivities must be non-positive")
    cand = t.empty_like(rho)
    fb = t.empty_like(rho)
    fp = t.empty_like(rho)

    def volumes(lams):
        out = []
        for lam in lams:
            _lib.call("tf_oc_apply_f64", n, D.ptr(rho), D.ptr(dc), D.ptr(dv), float(s.move), 0.5, float(lam),
                      D.ptr(cand), st)
            _lib.call("tf_filter_grid_f64", ctypes_ref(grid), float(rmin), D.ptr(inv_rs), D.ptr(cand),
                      D.ptr(fb), 0, st)
            _lib.call("tf_project_f64", n, float(s.beta), 0.5, D.ptr(fb), D.ptr(fp), None, st)
            _lib.call("tf_stats_f64", n, None, None, None, D.ptr(fp), D.ptr(work), D.ptr(stats), st)
            out.append(float(stats[2].item()) / n)
        return out

    res = oc_bisect(volumes, vf, batch=1)
    if res.status == "stalled":
        raise RuntimeError(f"OC bisection stalled with volume error {res.best_err:.3e}")
    _lib.call("tf_oc_apply_f64", n, D.ptr(rho), D.ptr(dc), D.ptr(dv), float(s.move), 0.5, float(res.lam),
              D.ptr(rho_new), st)


def run_simp_device(problem, config, schedule):
    from .simp import IterationRecord, SelectedRecord, SimpResult

    t = D.torch()
    dev = D.require_cuda()
    t_start = time.perf_counter()
    mesh, bcs = problem.mesh, problem.bcs
    n = mesh.n_elem
    prec = get_precision(config.precision)
    dt = prec.dtype
    # the (immutable) mesh's connectivity is cached on the mesh object, so a
    # repeated run on the same problem reuses its device problem, PCG handle
    # and tuned launch shapes instead of rebuilding them in iteration 1
    edof = D.CACHE.get(mesh, "edof", lambda: build_edof(mesh))
    grid = _lib.tf_grid(mesh.nelx, mesh.nely, mesh.nelz)
    st = D.stream_ptr()
    f64 = t.float64

    # operator shell: connectivity/constraints uploaded once, scale set per iteration
    op = MatFreeOperator(mesh, edof, bcs, np.ones(n), SimpParams(3.0), prec,
                         variant=config.variant, scatter=config.scatter, nu=config.nu,
                         backend=config.backend, grid_kernel=config.grid_kernel)
    if not op.structured or config.variant != "fused":
        raise ValueError("device SIMP path needs the fused structured operator")
    sfx = "f64" if np.dtype(dt) == np.float64 else "f32"

    rho = t.full((n,), problem.volume_fraction, dtype=f64, device=dev)
    rho_bar = t.empty_like(rho)
    rho_phys = t.empty_like(rho)
    dh = t.empty_like(rho)
    sens = t.empty_like(rho)
    dc = t.empty_like(rho)
    rho_new = t.empty_like(rho)
    inv_rs = t.empty_like(rho)
    f_dev = t.as_tensor(np.asarray(bcs.force, dtype=np.float64), device=dev)
    # the load vector, uploaded once (device_pcg would copy a host array per solve)
    rhs = D.to_dev(np.ascontiguousarray(bcs.force, dtype=dt), dt)
    work = t.empty(int(_lib.load().tf_work_doubles(max(n, mesh.n_dof))), dtype=f64, device=dev)
    stats = t.empty(3, dtype=f64, device=dev)
    bad = t.zeros(1, dtype=t.int32, device=dev)
    oc_rep_dev = t.zeros(4, dtype=f64, device=dev)  # tf_oc_report is 24 bytes
    oc_rep = _lib.tf_oc_report()

    def build_filter(rmin):
        _lib.call("tf_filter_rowsum_f64", ctypes_ref(grid), float(rmin), D.ptr(inv_rs), st)

    rmin_built = schedule.at(1).rmin
    build_filter(rmin_built)
    u_warm = None
    selected = None
    restarts = 0
    history = []
    total_cg = 0

    for it in range(1, schedule.total_iterations + 1):
        t_it = time.perf_counter()
        s = schedule.at(it)
        if abs(s.rmin - rmin_built) >= config.filter_rebuild_delta:
            rmin_built = s.rmin
            build_filter(rmin_built)
        _lib.call("tf_filter_grid_f64", ctypes_ref(grid), float(rmin_built), D.ptr(inv_rs),
                  D.ptr(rho), D.ptr(rho_bar), 0, st)
        _lib.call("tf_project_f64", n, float(s.beta), 0.5, D.ptr(rho_bar), D.ptr(rho_phys),
                  D.ptr(dh), st)
        _lib.call(f"tf_simp_scale_{sfx}", n, float(s.p), RHO_MIN, D.ptr(rho_phys),
                  D.ptr(op._scale_dev), D.ptr(bad), st)
        op.simp = SimpParams(p=s.p)
        diag_d, _ = op.diagonal_device()
        x0 = u_warm if (config.warm_start and u_warm is not None) else None
        u_d, rep = device_pcg(op, rhs, diag_d, config.cg, x0=x0, return_device=True)
        total_cg += rep.iterations
        u64 = u_d.double()
        _lib.call("tf_stats_f64", mesh.n_dof, D.ptr(f_dev), D.ptr(u64), None, None,
                  D.ptr(work), D.ptr(stats), st)
        c = float(stats[0].item())
        _lib.call("tf_stats_f64", n, None, None, D.ptr(rho_phys), None, D.ptr(work), D.ptr(stats), st)
        g = 4.0 * float(stats[1].item()) / n

        if s.p >= config.select_p_min and g < config.select_gray_max and (
                selected is None or c < selected.compliance):
            selected = _Selected(it, c, g, rho.clone(), rho_phys.clone(), u64.clone(), s.p, s.beta)

        restarted = False
        if selected is not None and c > config.restart_threshold * selected.compliance:
            rho = selected.rho.clone()
            u_warm = selected.u.to(u_d.dtype)
            restarts += 1
            restarted = True
        else:
            u_warm = u_d
            energies = op.energies_device(u64)
            _lib.call("tf_sensitivity_f64", n, float(s.p), RHO_MIN, D.ptr(rho_phys),
                      D.ptr(energies), D.ptr(dh), D.ptr(sens), st)
            _lib.call("tf_filter_grid_f64", ctypes_ref(grid), float(rmin_built), D.ptr(inv_rs),
                      D.ptr(sens), D.ptr(dc), 1, st)
            if config.volume_on == "raw":
                _lib.call("tf_oc_update_f64", n, D.ptr(rho), D.ptr(dc), None,
                          float(problem.volume_fraction), float(s.move), 1e-6, 0.5, 200,
                          D.ptr(rho_new), D.ptr(work), D.ptr(oc_rep_dev), st)
                rep_host = oc_rep_dev.cpu().numpy()
                ctypes.memmove(ctypes.addressof(oc_rep), rep_host.ctypes.data, ctypes.sizeof(oc_rep))
                status = _lib.OC_STATUS[oc_rep.status]
                if status == "bad_input":
                    raise ValueError("compliance sensitivities must be non-positive")
                if status == "stalled":
                    raise RuntimeError(f"OC bisection stalled with volume error {oc_rep.best_err:.3e}")
            else:
                _oc_projected(n, grid, rmin_built, inv_rs, rho, dc, dh, s, problem.volume_fraction,
                              rho_new, work, stats, st)
            rho, rho_new = rho_new, rho
        if int(bad.item()):
            raise ValueError("densities must lie in [0, 1]")
        _lib.call("tf_stats_f64", n, None, None, None, D.ptr(rho), D.ptr(work), D.ptr(stats), st)
        vol = float(stats[2].item()) / n
        history.append(IterationRecord(it, c, g, rep.iterations, rep.converged, s.p, s.beta,
                                       s.move, s.rmin, vol, restarted, time.perf_counter() - t_it))

    fin = schedule.at(schedule.total_iterations)
    _lib.call("tf_filter_grid_f64", ctypes_ref(grid), float(rmin_built), D.ptr(inv_rs),
              D.ptr(rho), D.ptr(rho_bar), 0, st)
    _lib.call("tf_project_f64", n, float(fin.beta), 0.5, D.ptr(rho_bar), D.ptr(rho_phys), None, st)
    sel = None
    if selected is not None:
        sel = SelectedRecord(selected.iteration, selected.compliance, selected.grayness,
                             selected.rho.cpu().numpy(), selected.rho_phys.cpu().numpy(),
                             selected.u.cpu().numpy(), selected.p, selected.beta)
    return SimpResult(history, sel, restarts, rho.cpu().numpy(), rho_phys.cpu().numpy(), total_cg,
                      time.perf_counter() - t_start, config, problem.name)
