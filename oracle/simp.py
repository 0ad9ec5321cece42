"""TEST INFRASTRUCTURE ONLY -- CPU restatement of the reference SIMP loop.

Only tests/ and bench.py (cpu_baseline leg, ``--impl reference``) may import
this module; the product package never does.  It restates
``/root/reference/pkg/src/topofuse/simp.py`` for the raw-volume path:

  * build_cone_filter (simp.py:33-69): row-stochastic cone weights
    max(0, rmin - dist) as a scipy CSR, rows normalised;
  * heaviside_projection / derivative (simp.py:72-84), grayness (:87-91);
  * compliance_sensitivity + chain_to_design (simp.py:96-108) on the oracle's
    element energies (_kernels_numba.py:241-256);
  * oc_update (simp.py:111-175): bracket by halving/doubling, bisection to
    |mean - V_f| <= 1e-6;
  * run_simp (simp.py:324-448): schedule state, filter rebuild rule, warm
    start, selection gate and 1.12x restart rule, one OC step per iteration,

with every equilibrium solve through the oracle's C port of the fused kernels
(oracle.apply, serial or OpenMP atomic scatter) and its restated PCG
(oracle.pcg).  Pinned against the reference's own c1 trajectory
(tests/golden/simp_c1_fp64.npz) in tests/test_oracle.py.
"""

from __future__ import annotations

import time

import numpy as np
import scipy.sparse as sp

from . import apply, diagonal, element_energies, pcg

HEAVISIDE_ETA = 0.5
RHO_MIN = 1e-9


def cone_filter(nelx, nely, nelz, rmin):
    """simp.py:33-69: weights over all offsets within the radius, CSR, rows normalised."""
    ids = np.arange(nelx * nely * nelz, dtype=np.int64).reshape(nelz, nely, nelx)
    reach = int(np.ceil(rmin))
    rows, cols, vals = [], [], []
    for dk in range(-reach, reach + 1):
        for dj in range(-reach, reach + 1):
            for di in range(-reach, reach + 1):
                wgt = rmin - np.sqrt(di * di + dj * dj + dk * dk)
                if wgt <= 0.0:
                    continue
                zs, ys, xs = (slice(max(0, -d), n - max(0, d)) for d, n in ((dk, nelz), (dj, nely), (di, nelx)))
                zd, yd, xd = (slice(max(0, d), n + min(0, d)) for d, n in ((dk, nelz), (dj, nely), (di, nelx)))
                src, dst = ids[zs, ys, xs], ids[zd, yd, xd]
                rows.append(dst.ravel())
                cols.append(src.ravel())
                vals.append(np.full(src.size, wgt))
    n = nelx * nely * nelz
    w = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(n, n)).tocsr()
    return sp.diags(1.0 / np.asarray(w.sum(axis=1)).ravel()) @ w


def heaviside(x, beta, eta=HEAVISIDE_ETA):
    d = np.tanh(beta * eta) + np.tanh(beta * (1.0 - eta))
    return (np.tanh(beta * eta) + np.tanh(beta * (x - eta))) / d


def heaviside_deriv(x, beta, eta=HEAVISIDE_ETA):
    d = np.tanh(beta * eta) + np.tanh(beta * (1.0 - eta))
    return beta / (np.cosh(beta * (x - eta)) ** 2 * d)


def oc_step(rho, dc, dv, vf, move, vol_tol=1e-6, damping=0.5, max_bisect=200):
    """simp.py:111-175 with the raw-mean volume."""
    if np.any(dc > 1e-12):
        raise ValueError("compliance sensitivities must be non-positive")
    lower, upper = np.maximum(0.0, rho - move), np.minimum(1.0, rho + move)
    ratio = -dc / dv

    def cand(lam):
        return np.clip(rho * (ratio / lam) ** damping, lower, upper)

    lo = hi = 1.0
    for _ in range(200):
        if float(np.mean(cand(lo))) >= vf:
            break
        lo *= 0.5
    else:
        return cand(lo)
    for _ in range(200):
        if float(np.mean(cand(hi))) <= vf:
            break
        hi *= 2.0
    else:
        return cand(hi)
    best = None
    for _ in range(max_bisect):
        lam = 0.5 * (lo + hi)
        c = cand(lam)
        err = abs(float(np.mean(c)) - vf)
        if best is None or err < best[0]:
            best = (err, c)
        if err <= vol_tol:
            return c
        if float(np.mean(c)) > vf:
            lo = lam
        else:
            hi = lam
    if best[0] <= vol_tol:
        return best[1]
    raise RuntimeError(f"OC bisection stalled with volume error {best[0]:.3e}")


def schedule_state(phases, rmin_start, it):
    """ContinuationSchedule.at (simp.py:220-234); phases: (start, end, p, beta, move, rmin_end)."""
    rmin_in = rmin_start
    for start, end, p, beta, move, rmin_end in phases:
        if it <= end:
            rmin = rmin_end if end == start else rmin_in + (rmin_end - rmin_in) * (it - start) / (end - start)
            return p, beta, move, rmin
        rmin_in = rmin_end
    raise ValueError("iteration outside schedule")


def run_simp(dims, edof, fixed_dofs, force, vf, phases, rmin_start, ke64, precision="fp64",
             scatter="serial", iterations=None, rel_tol=1e-5, max_iter=1000, recompute_every=50,
             restart_threshold=1.12, select_p_min=3.0, select_gray_max=0.25, rebuild_delta=0.05):
    """simp.py:324-448 (raw volume, warm start).  Returns per-iteration records."""
    nelx, nely, nelz = dims
    n_elem = nelx * nely * nelz
    n_dof = force.size
    dt = np.float64 if precision == "fp64" else np.float32
    ke = np.ascontiguousarray(ke64, dtype=dt)
    total = phases[-1][1] if iterations is None else iterations
    rho = np.full(n_elem, vf)
    rmin_built = schedule_state(phases, rmin_start, 1)[3]
    filt = cone_filter(nelx, nely, nelz, rmin_built)
    u_warm, selected, hist = None, None, []
    for it in range(1, total + 1):
        t0 = time.perf_counter()
        p, beta, move, rmin = schedule_state(phases, rmin_start, it)
        if abs(rmin - rmin_built) >= rebuild_delta:
            filt, rmin_built = cone_filter(nelx, nely, nelz, rmin), rmin
        rho_bar = filt @ rho
        rho_phys = heaviside(rho_bar, beta)
        scale = (RHO_MIN + (1.0 - RHO_MIN) * np.clip(rho_phys, 0.0, 1.0) ** p).astype(dt)
        A = lambda x: apply(edof, ke, scale, x, fixed_dofs, n_dof, "fused", scatter)  # noqa: E731
        x0 = None if u_warm is None else np.ascontiguousarray(u_warm, dtype=dt)
        u, info = pcg(A, np.ascontiguousarray(force, dtype=dt), diagonal(edof, ke, scale, fixed_dofs, n_dof),
                      rel_tol, max_iter, recompute_every, x0=x0)
        c = float(np.dot(np.asarray(force, np.float64), np.asarray(u, np.float64)))
        g = float(4.0 * np.mean(rho_phys * (1.0 - rho_phys)))
        if p >= select_p_min and g < select_gray_max and (selected is None or c < selected[0]):
            selected = (c, rho.copy(), np.asarray(u, np.float64).copy())
        restarted = selected is not None and c > restart_threshold * selected[0]
        if restarted:
            rho, u_warm = selected[1].copy(), selected[2].copy()
        else:
            u_warm = np.asarray(u, np.float64)
            energies = element_energies(edof, ke64, u_warm)
            dc_phys = -(p * (1.0 - RHO_MIN) * np.clip(rho_phys, 0.0, 1.0) ** (p - 1.0)) * energies
            dc = filt.T @ (heaviside_deriv(rho_bar, beta) * dc_phys)
            rho = oc_step(rho, dc, np.ones(n_elem), vf, move)
        hist.append({"iteration": it, "compliance": c, "grayness": g, "cg_iterations": info["iterations"],
                     "restarted": restarted, "volume": float(np.mean(rho)), "wall_s": time.perf_counter() - t0})
    return hist, rho
