"""x-slab distributed SIMP loop (reference simp.py:324-448 over P GPUs).

SURVEY 8e: the headline metric is SIMP seconds per iteration at 1/2/4/8 B200.
Every rank owns the element layers [x0, x1) of its slab (slab.py) and runs the
same continuation loop as ``simp_device.run_simp_device`` on them:

  filter / projection   the cone filter reaches ``ceil(rmin)`` layers; each
                        rank extends its slab by H = 2 ceil(rmin) element
                        layers on every interior side (halo P2P), builds the
                        row sums on the extended grid and keeps its own
                        layers.  Owned outputs of F and F^T then sum exactly
                        the neighbours and row sums the single-GPU filter
                        sums (rows within H/2 of the halo edge are complete),
                        in the same stencil order -- bitwise the one-GPU
                        filter.
  equilibrium           ``slab.slab_pcg`` on the slab operator (interface
                        partial-sum exchange, owner-computes dots).
  scalars               compliance, grayness, volume: rank-local fixed-order
                        sums, all-gathered and added in rank order, so every
                        rank takes identical selection/restart decisions.
  OC                    the bracket/bisection of simp.py:111-175 runs on the
                        host over global volumes; each round trip evaluates up
                        to 15 multipliers on the device (tf_oc_volumes_f64):
                        8 bracket steps, or the next 4 bisection levels (all
                        15 nodes of the subtree), then walks the reference's
                        sequence over them -- same multipliers, same stop
                        rule, ~4x fewer all-gathers.

Differences from one GPU are summation order only (CG dots, scalar sums,
interface partials), so histories agree to rounding and CG counts to +-1.
"""

from __future__ import annotations

import math
import time

import numpy as np

from .element import RHO_MIN, SimpParams
from .mesh import StructuredMesh
from .slab import SlabOperator, SlabPartition, gpu_local_kernels, slab_pcg

OC_MAX_LAMS = 15


# -- global sums --------------------------------------------------------------------


def rank_sum(vals, group=None):
    """Sum of a small FP64 vector over ranks, added in rank order (every rank
    gets the bitwise-same result).  `vals`: torch tensor on any device."""
    import torch
    import torch.distributed as dist

    t = vals.detach().to(torch.float64).reshape(-1)
    if not (dist.is_initialized() and dist.get_world_size(group) > 1):
        return t.cpu().numpy().copy()
    ws = dist.get_world_size(group)
    if dist.get_backend(group) == "gloo":
        t = t.cpu()
    parts = [torch.empty_like(t) for _ in range(ws)]
    dist.all_gather(parts, t.contiguous(), group=group)
    acc = parts[0].cpu().numpy().copy()
    for p in parts[1:]:
        acc = acc + p.cpu().numpy()
    return acc


# -- OC bisection over a global volume function ------------------------------------


class OcOutcome:
    def __init__(self, lam, status, evaluations, best_err):
        self.lam, self.status, self.evaluations, self.best_err = lam, status, evaluations, best_err


def oc_bisect(volumes, volume_fraction, vol_tol=1e-6, max_bisect=200, batch=OC_MAX_LAMS):
    """Multiplier selection of oc_update (simp.py:111-175) over `volumes(lams)
    -> list of global mean volumes`, evaluating up to `batch` multipliers per
    call.  Returns the multiplier whose candidate the reference returns; the
    evaluated sequence is the reference's (the batch only adds speculative
    evaluations off its path).  status: ok | saturated | stalled."""
    vf = volume_fraction
    evals = 0
    nb = max(1, min(8, batch))
    # bracket from below: lam_lo = 0.5^k
    lam_lo, found, k = 1.0, False, 0
    while k < 200 and not found:
        lams = [0.5 ** (k + q) for q in range(min(nb, 200 - k))]
        vols = volumes(lams)
        for lam, v in zip(lams, vols):
            evals += 1
            k += 1
            if v >= vf:
                lam_lo, found = lam, True
                break
    if not found:
        return OcOutcome(0.5 ** 200, "saturated", evals, None)
    lam_hi, found, k = 1.0, False, 0
    while k < 200 and not found:
        lams = [2.0 ** (k + q) for q in range(min(nb, 200 - k))]
        vols = volumes(lams)
        for lam, v in zip(lams, vols):
            evals += 1
            k += 1
            if v <= vf:
                lam_hi, found = lam, True
                break
    if not found:
        return OcOutcome(2.0 ** 200, "saturated", evals, None)
    depth = max(1, int(math.log2(batch + 1)))
    best_err, best_lam, b = None, None, 0
    while b < max_bisect:
        # the next `depth` levels of the bisection tree under (lam_lo, lam_hi)
        levels = min(depth, max_bisect - b)
        nodes = {}
        frontier = [((), lam_lo, lam_hi)]
        for _ in range(levels):
            nxt = []
            for path, lo, hi in frontier:
                mid = 0.5 * (lo + hi)
                nodes[path] = mid
                nxt += [(path + (1,), mid, hi), (path + (0,), lo, mid)]
            frontier = nxt
        keys = list(nodes)
        vols = dict(zip(keys, volumes([nodes[p] for p in keys])))
        path = ()
        for _ in range(levels):
            lam, v = nodes[path], vols[path]
            b += 1
            evals += 1
            err = abs(v - vf)
            if best_err is None or err < best_err:
                best_err, best_lam = err, lam
            if err <= vol_tol:
                return OcOutcome(lam, "ok", evals, best_err)
            # v > vf: too much material -> raise lam (right child keeps hi)
            if v > vf:
                lam_lo, path = lam, path + (1,)
            else:
                lam_hi, path = lam, path + (0,)
    status = "ok" if best_err <= vol_tol else "stalled"
    return OcOutcome(best_lam, status, evals, best_err)


# -- element-layer halos ------------------------------------------------------------


class ElementHalo:
    """Extends a slab's per-element field by `h` element layers on each
    interior side (x-neighbours' edge layers), for the cone filter."""

    def __init__(self, part: SlabPartition, h: int, device, group=None):
        lm = part.local_mesh
        if (part.has_left or part.has_right) and lm.nelx < h:
            raise ValueError(f"slab of {lm.nelx} element layers is thinner than the filter halo {h}")
        self.part, self.h, self.group, self.device = part, h, group, device
        self.hl = h if part.has_left else 0
        self.hr = h if part.has_right else 0
        self.mesh = StructuredMesh(lm.nelx + self.hl + self.hr, lm.nely, lm.nelz)
        self.shape = (lm.nelz, lm.nely, lm.nelx)

    def extend(self, f):
        import torch
        import torch.distributed as dist

        p, h = self.part, self.h
        v = f.view(self.shape)
        if not (p.has_left or p.has_right):
            return f.clone()
        host = f.is_cuda and dist.get_backend(self.group) == "gloo"
        ops, recv_l, recv_r = [], None, None
        mk = (lambda t: t.cpu()) if host else (lambda t: t)
        if p.has_left:
            send_l = mk(v[..., :h].contiguous())
            recv_l = torch.empty_like(send_l)
            ops += [dist.P2POp(dist.isend, send_l, p.rank - 1, self.group),
                    dist.P2POp(dist.irecv, recv_l, p.rank - 1, self.group)]
        if p.has_right:
            send_r = mk(v[..., v.shape[2] - h:].contiguous())
            recv_r = torch.empty_like(send_r)
            ops += [dist.P2POp(dist.isend, send_r, p.rank + 1, self.group),
                    dist.P2POp(dist.irecv, recv_r, p.rank + 1, self.group)]
        for w in dist.batch_isend_irecv(ops):
            w.wait()
        cat = [t.to(f.device) for t in (recv_l,) if t is not None] + [v] + \
              [t.to(f.device) for t in (recv_r,) if t is not None]
        return torch.cat(cat, dim=2).reshape(-1).contiguous()

    def owned(self, fext):
        nz, ny, nx = self.shape
        if self.hl == 0 and self.hr == 0:
            return fext.clone()  # never alias the caller's scratch buffer
        return fext.view(nz, ny, nx + self.hl + self.hr)[..., self.hl:self.hl + nx].reshape(-1).contiguous()


# -- the loop ----------------------------------------------------------------------


def _gather_elem(part, local, group):
    """Global per-element array (numpy) from every rank's slab (all ranks)."""
    import torch.distributed as dist

    pieces = [None] * dist.get_world_size(group) if dist.is_initialized() else None
    mine = (part.local_elem_to_global(), local.cpu().numpy())
    if pieces is None:
        pieces = [mine]
    else:
        dist.all_gather_object(pieces, mine, group=group)
    out = np.empty(part.mesh.n_elem)
    for idx, val in pieces:
        out[idx] = val
    return out


def _gather_dof(part, local, group):
    import torch.distributed as dist

    pieces = [None] * dist.get_world_size(group) if dist.is_initialized() else None
    mine = (part.local_dof_to_global(), local.cpu().numpy())
    if pieces is None:
        pieces = [mine]
    else:
        dist.all_gather_object(pieces, mine, group=group)
    out = np.empty(part.mesh.n_dof)
    for idx, val in pieces:
        out[idx] = val
    return out


def slab_run_simp(problem, config=None, group=None, device=None, gather: bool = True):
    """Distributed continuation SIMP on the x-slab decomposition (see
    _slab_run_simp); runs with Python's automatic cyclic GC paused."""
    from . import _device as D

    with D.gc_paused():
        return _slab_run_simp(problem, config, group, device, gather)


def _slab_run_simp(problem, config=None, group=None, device=None, gather: bool = True):
    """Distributed continuation SIMP on the x-slab decomposition.

    Same loop, schedule, selection/restart rules and raw-volume OC as
    ``simp.run_simp`` (device path); returns a ``SimpResult`` whose history
    holds the global scalars (identical on every rank).  With ``gather`` the
    result's fields are assembled to global arrays on every rank.
    """
    import torch
    import torch.distributed as dist

    from . import _device as D
    from . import _lib
    from .operator import ctypes_ref
    from .precision import get_precision
    from .simp import IterationRecord, SelectedRecord, SimpConfig, SimpResult, default_schedule

    config = config or SimpConfig()
    if config.variant != "fused":
        raise ValueError("slab SIMP runs the fused operator")
    schedule = config.schedule or default_schedule()
    t_start = time.perf_counter()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    dev = device or D.require_cuda()
    mesh, bcs = problem.mesh, problem.bcs
    part = SlabPartition(mesh, world, rank)
    lm = part.local_mesh
    n, n_glob = lm.n_elem, mesh.n_elem
    prec = get_precision(config.precision)
    dt = D.tdtype(prec.dtype)
    f64 = torch.float64
    sfx = "f64" if np.dtype(prec.dtype) == np.float64 else "f32"
    st = D.stream_ptr()

    rmax = max([schedule.rmin_start] + [ph.rmin_end for ph in schedule.phases])
    if rmax > 3.0:
        raise ValueError("slab SIMP supports filter radii <= 3")
    halo = ElementHalo(part, 2 * int(math.ceil(rmax)), dev, group)
    ext_grid = _lib.tf_grid(halo.mesh.nelx, halo.mesh.nely, halo.mesh.nelz)

    bcs_l = part.local_bcs(bcs)
    op_l, local_apply, local_diag = gpu_local_kernels(part, bcs_l, np.ones(n), SimpParams(3.0),
                                                      config.precision, nu=config.nu)
    sop = SlabOperator(part, bcs_l, local_apply, local_diag, dev, dt, group)
    owned = sop.owned
    b = torch.as_tensor(np.asarray(bcs_l.force), dtype=dt, device=dev)
    f_loc = torch.as_tensor(np.asarray(bcs_l.force), dtype=f64, device=dev)

    rho = torch.full((n,), problem.volume_fraction, dtype=f64, device=dev)
    rho_bar = torch.empty_like(rho)
    rho_phys = torch.empty_like(rho)
    dh = torch.empty_like(rho)
    sens = torch.empty_like(rho)
    rho_new = torch.empty_like(rho)
    inv_rs = torch.empty(halo.mesh.n_elem, dtype=f64, device=dev)
    y_ext = torch.empty_like(inv_rs)
    bad = torch.zeros(1, dtype=torch.int32, device=dev)
    oc_work = torch.empty(int(_lib.load().tf_oc_work_doubles(n)), dtype=f64, device=dev)
    oc_sums = torch.empty(OC_MAX_LAMS + 1, dtype=f64, device=dev)

    def build_filter(rmin):
        _lib.call("tf_filter_rowsum_f64", ctypes_ref(ext_grid), float(rmin), D.ptr(inv_rs), st)

    def filt(x, rmin, transpose):
        xe = halo.extend(x)
        _lib.call("tf_filter_grid_f64", ctypes_ref(ext_grid), float(rmin), D.ptr(inv_rs), D.ptr(xe),
                  D.ptr(y_ext), int(transpose), st)
        return halo.owned(y_ext)

    def scalars(c_local, gray_local, vol_local):
        return rank_sum(torch.stack([c_local, gray_local, vol_local]), group)

    rmin_built = schedule.at(1).rmin
    build_filter(rmin_built)
    u_warm = None
    selected = None
    restarts = 0
    history = []
    total_cg = 0
    last_oc = None

    for it in range(1, schedule.total_iterations + 1):
        t_it = time.perf_counter()
        s = schedule.at(it)
        if abs(s.rmin - rmin_built) >= config.filter_rebuild_delta:
            rmin_built = s.rmin
            build_filter(rmin_built)
        rho_bar = filt(rho, rmin_built, 0)
        _lib.call("tf_project_f64", n, float(s.beta), 0.5, D.ptr(rho_bar), D.ptr(rho_phys), D.ptr(dh), st)
        _lib.call(f"tf_simp_scale_{sfx}", n, float(s.p), RHO_MIN, D.ptr(rho_phys),
                  D.ptr(op_l._scale_dev), D.ptr(bad), st)
        diag = sop.diagonal()
        x0 = u_warm if (config.warm_start and u_warm is not None) else None
        u, info = slab_pcg(sop, b, diag, rel_tol=config.cg.rel_tol, max_iter=config.cg.max_iter,
                           recompute_every=config.cg.recompute_every, x0=x0)
        total_cg += info["iterations"]
        u64 = u.double()
        cgf = torch.sum(f_loc[owned] * u64[owned])
        gray = torch.sum(rho_phys * (1.0 - rho_phys))
        c, gsum, _ = scalars(cgf, gray, torch.zeros((), dtype=f64, device=dev))
        c, g = float(c), 4.0 * float(gsum) / n_glob

        if s.p >= config.select_p_min and g < config.select_gray_max and (
                selected is None or c < selected[1]):
            selected = (it, c, g, rho.clone(), rho_phys.clone(), u64.clone(), s.p, s.beta)

        restarted = False
        if selected is not None and c > config.restart_threshold * selected[1]:
            rho = selected[3].clone()
            u_warm = selected[5].to(dt)
            restarts += 1
            restarted = True
        else:
            u_warm = u
            energies = op_l.energies_device(u64)
            _lib.call("tf_sensitivity_f64", n, float(s.p), RHO_MIN, D.ptr(rho_phys),
                      D.ptr(energies), D.ptr(dh), D.ptr(sens), st)
            dc = filt(sens, rmin_built, 1)
            checked = [False]
            dv = None
            if config.volume_on == "projected":
                # dv = max(F^T dh, 1e-12); volumes are projected means
                # (simp.py:393-401): per multiplier one candidate, one halo
                # exchange + filter, one projection, one rank sum
                dv = filt(dh, rmin_built, 1).clamp_(min=1e-12)
                if float(rank_sum((dc > 1e-12).sum().double().reshape(1), group)[0]) > 0:
                    raise ValueError("compliance sensitivities must be non-positive")
                cand, fp = torch.empty_like(rho), torch.empty_like(rho)

            def volumes(lams):
                if dv is not None:
                    out = []
                    for lam in lams:
                        _lib.call("tf_oc_apply_f64", n, D.ptr(rho), D.ptr(dc), D.ptr(dv), float(s.move), 0.5,
                                  float(lam), D.ptr(cand), st)
                        fb = filt(cand, rmin_built, 0)
                        _lib.call("tf_project_f64", n, float(s.beta), 0.5, D.ptr(fb), D.ptr(fp), None, st)
                        out.append(float(rank_sum(torch.sum(fp).reshape(1), group)[0]) / n_glob)
                    return out
                lam_arr = np.asarray(lams, dtype=np.float64)  # alive across the call
                _lib.call("tf_oc_volumes_f64", n, D.ptr(rho), D.ptr(dc), None, float(s.move), 0.5,
                          lam_arr.ctypes.data, len(lams), D.ptr(oc_sums), D.ptr(oc_work), st)
                tot = rank_sum(oc_sums, group)
                if not checked[0]:
                    if tot[OC_MAX_LAMS] > 0:
                        raise ValueError("compliance sensitivities must be non-positive")
                    checked[0] = True
                return [float(v) / n_glob for v in tot[:len(lams)]]

            last_oc = oc_bisect(volumes, problem.volume_fraction, batch=1 if dv is not None else OC_MAX_LAMS)
            if last_oc.status == "stalled":
                raise RuntimeError(f"OC bisection stalled with volume error {last_oc.best_err:.3e}")
            _lib.call("tf_oc_apply_f64", n, D.ptr(rho), D.ptr(dc), D.ptr(dv) if dv is not None else None,
                      float(s.move), 0.5, float(last_oc.lam), D.ptr(rho_new), st)
            rho, rho_new = rho_new, rho
        if int(rank_sum(bad.double(), group)[0]):
            raise ValueError("densities must lie in [0, 1]")
        vol = float(rank_sum(torch.sum(rho).reshape(1), group)[0]) / n_glob
        history.append(IterationRecord(it, c, g, info["iterations"], info["termination"] == "converged",
                                       s.p, s.beta, s.move, s.rmin, vol, restarted,
                                       time.perf_counter() - t_it))

    fin = schedule.at(schedule.total_iterations)
    rho_bar = filt(rho, rmin_built, 0)
    _lib.call("tf_project_f64", n, float(fin.beta), 0.5, D.ptr(rho_bar), D.ptr(rho_phys), None, st)
    wall = time.perf_counter() - t_start
    if not gather:
        sel = None
        if selected is not None:
            sel = SelectedRecord(selected[0], selected[1], selected[2], selected[3].cpu().numpy(),
                                 selected[4].cpu().numpy(), selected[5].cpu().numpy(), selected[6], selected[7])
        return SimpResult(history, sel, restarts, rho.cpu().numpy(), rho_phys.cpu().numpy(), total_cg,
                          wall, config, problem.name)
    sel = None
    if selected is not None:
        sel = SelectedRecord(selected[0], selected[1], selected[2], _gather_elem(part, selected[3], group),
                             _gather_elem(part, selected[4], group), _gather_dof(part, selected[5], group),
                             selected[6], selected[7])
    return SimpResult(history, sel, restarts, _gather_elem(part, rho, group), _gather_elem(part, rho_phys, group),
                      total_cg, wall, config, problem.name)


__all__ = ["ElementHalo", "OcOutcome", "oc_bisect", "rank_sum", "slab_run_simp"]
