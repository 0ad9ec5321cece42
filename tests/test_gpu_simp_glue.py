"""GPU parity of the device SIMP glue (filter, projection, sensitivity, OC)
against the host restatements of the reference (simp.py:33-175)."""

from __future__ import annotations

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _dev(a):
    import torch

    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device="cuda")


@pytest.mark.parametrize("dims,rmin", [((7, 5, 4), 1.5), ((12, 6, 6), 1.35), ((5, 5, 5), 2.2),
                                       ((30, 10, 8), 1.2)])
def test_filter_and_transpose_match_scipy(dims, rmin):
    import torch

    from paper_2604_18020_b200 import _device as D
    from paper_2604_18020_b200 import _lib
    from paper_2604_18020_b200.mesh import StructuredMesh
    from paper_2604_18020_b200.operator import ctypes_ref
    from paper_2604_18020_b200.simp import build_cone_filter

    m = StructuredMesh(*dims)
    F = build_cone_filter(m, rmin)
    rng = np.random.default_rng(4)
    x = rng.uniform(0, 1, m.n_elem)
    g = _lib.tf_grid(*dims)
    inv = torch.empty(m.n_elem, dtype=torch.float64, device="cuda")
    y = torch.empty_like(inv)
    _lib.call("tf_filter_rowsum_f64", ctypes_ref(g), rmin, D.ptr(inv), D.stream_ptr())
    xd = _dev(x)
    for tr, want in ((0, F @ x), (1, F.T @ x)):
        _lib.call("tf_filter_grid_f64", ctypes_ref(g), rmin, D.ptr(inv), D.ptr(xd), D.ptr(y), tr,
                  D.stream_ptr())
        assert np.abs(y.cpu().numpy() - want).max() <= 1e-14 * np.abs(want).max()


def test_projection_and_sensitivity():
    import torch

    from paper_2604_18020_b200 import _device as D
    from paper_2604_18020_b200 import _lib
    from paper_2604_18020_b200.element import SimpParams, simp_scale_derivative
    from paper_2604_18020_b200.simp import heaviside_derivative, heaviside_projection

    rng = np.random.default_rng(5)
    rb = rng.uniform(0, 1, 5000)
    e = rng.uniform(0, 2, 5000)
    for beta in (1.0, 4.0, 16.0, 32.0):
        rp = torch.empty(5000, dtype=torch.float64, device="cuda")
        dh = torch.empty_like(rp)
        rb_d, e_d = _dev(rb), _dev(e)
        _lib.call("tf_project_f64", 5000, beta, 0.5, D.ptr(rb_d), D.ptr(rp), D.ptr(dh), D.stream_ptr())
        np.testing.assert_allclose(rp.cpu().numpy(), heaviside_projection(rb, beta), rtol=1e-13, atol=1e-15)
        np.testing.assert_allclose(dh.cpu().numpy(), heaviside_derivative(rb, beta), rtol=1e-12)
        out = torch.empty_like(rp)
        _lib.call("tf_sensitivity_f64", 5000, 3.0, 1e-9, D.ptr(rp), D.ptr(e_d), D.ptr(dh),
                  D.ptr(out), D.stream_ptr())
        want = heaviside_derivative(rb, beta) * (-simp_scale_derivative(heaviside_projection(rb, beta), SimpParams(3.0)) * e)
        np.testing.assert_allclose(out.cpu().numpy(), want, rtol=1e-12, atol=1e-12 * np.abs(want).max())


@pytest.mark.parametrize("n,vf,move", [(128, 0.4, 0.2), (10_000, 0.3, 0.05), (216_000, 0.3, 0.15),
                                        (10_000, 0.45, 0.1), (216_000, 0.5, 0.2), (50_000, 0.6, 0.02)])
def test_oc_update_matches_host(n, vf, move):
    import torch

    from paper_2604_18020_b200 import _device as D
    from paper_2604_18020_b200 import _lib
    from paper_2604_18020_b200.simp import oc_update

    rng = np.random.default_rng(n)
    rho = rng.uniform(0.05, 0.95, n)
    dc = -rng.uniform(0.01, 10.0, n)
    want = oc_update(rho, dc, np.ones(n), vf, move)
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    work = torch.empty(int(_lib.load().tf_work_doubles(n)), dtype=torch.float64, device="cuda")
    rep_d = torch.zeros(4, dtype=torch.float64, device="cuda")
    rho_d, dc_d = _dev(rho), _dev(dc)
    _lib.call("tf_oc_update_f64", n, D.ptr(rho_d), D.ptr(dc_d), None, vf, move, 1e-6, 0.5,
              200, D.ptr(out), D.ptr(work), D.ptr(rep_d), D.stream_ptr())
    rep = _lib.tf_oc_report()
    h = rep_d.cpu().numpy()
    ctypes.memmove(ctypes.addressof(rep), h.ctypes.data, ctypes.sizeof(rep))
    got = out.cpu().numpy()
    reachable = np.mean(np.maximum(0.0, rho - move)) <= vf <= np.mean(np.minimum(1.0, rho + move))
    # unreachable targets saturate at the nearest candidate, like simp.py:146-159
    assert _lib.OC_STATUS[rep.status] == ("ok" if reachable else "saturated")
    if reachable:
        assert abs(got.mean() - vf) <= 1e-6
    assert np.abs(got - want).max() <= 1e-9


def test_device_and_host_glue_agree_on_desk_problem():
    """Same algorithm, different reduction orders.  A single-phase (p=3, beta=1)
    schedule is not chaotic, so the two trajectories must agree tightly; the
    late beta=16..32 continuation phases amplify 1e-12 differences into
    neighbouring local optima (see test_gpu_solver.test_simp_desk_*)."""
    from paper_2604_18020_b200 import SimpConfig, make_preset, run_simp
    from paper_2604_18020_b200.simp import ContinuationSchedule, Phase

    pb = make_preset("cantilever", 0.2)
    sched = ContinuationSchedule((Phase(1, 30, p=3.0, beta=1.0, move=0.2, rmin_end=1.5),), 1.5)
    cfg = SimpConfig(schedule=sched, precision="fp64")
    a = run_simp(pb, cfg, device_glue=True)
    b = run_simp(pb, cfg, device_glue=False)
    ca = np.array([h.compliance for h in a.history])
    cb = np.array([h.compliance for h in b.history])
    np.testing.assert_allclose(ca, cb, rtol=1e-5)
    assert np.linalg.norm(a.rho_phys - b.rho_phys) <= 1e-5 * np.linalg.norm(b.rho_phys)
    assert [h.cg_iterations for h in a.history] == [h.cg_iterations for h in b.history] or \
        max(abs(x - y) for x, y in zip([h.cg_iterations for h in a.history],
                                       [h.cg_iterations for h in b.history])) <= 3
