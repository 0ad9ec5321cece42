"""GPU parity of the B200 operator kernels against the oracle and golden fixtures.

Tolerances are the reference's own (test_operator.py:41-78, north star):
FP64 max-abs <= 1e-12 * max|w|, FP32 <= 1e-5 * max|w|.  The exact grid variant
and the Jacobi diagonal must be BITWISE equal to the reference outputs.
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

import oracle
from conftest import load_golden, seeded_case

pytestmark = pytest.mark.gpu

TOL = {"fp64": 1e-12, "fp32": 1e-5}
SMALL = [((4, 3, 2), 11), ((5, 3, 2), 12), ((1, 1, 1), 1001), ((24, 12, 6), 42)]


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _op(m, edof, bcs, rho, prec, **kw):
    from paper_2604_18020_b200 import MatFreeOperator, SimpParams

    return MatFreeOperator(m, edof, bcs, rho, SimpParams(3.0), prec, **kw)


def _rel(got, want):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    return np.abs(got - want).max() / max(np.abs(want).max(), 1e-300)


@pytest.mark.parametrize("dims,seed", SMALL)
@pytest.mark.parametrize("prec", ["fp64", "fp32"])
@pytest.mark.parametrize("kernel", ["tile", "pull"])
def test_structured_fast_matches_reference(dims, seed, prec, kernel):
    g = load_golden(f"matvec_{'x'.join(map(str, dims))}.npz")
    m, edof, bcs, rho, v = seeded_case(dims, seed)
    op = _op(m, edof, bcs, rho, prec, grid_kernel=kernel)
    assert op.structured
    got = op.apply(v.astype(op.precision.dtype))
    assert _rel(got, g[f"apply_fused_{prec}"]) <= TOL[prec]
    assert np.array_equal(got[bcs.fixed_dofs], v.astype(op.precision.dtype)[bcs.fixed_dofs])


@pytest.mark.parametrize("dims,seed", SMALL)
@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_structured_exact_is_bitwise_reference(dims, seed, prec):
    g = load_golden(f"matvec_{'x'.join(map(str, dims))}.npz")
    m, edof, bcs, rho, v = seeded_case(dims, seed)
    op = _op(m, edof, bcs, rho, prec, exact=True)
    # unit_stiffness is the reference's Ke bitwise: nothing injected
    got = op.apply(v.astype(op.precision.dtype))
    assert np.array_equal(got, g[f"apply_fused_{prec}"])


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_full_size_c2_exact_hash_and_fast_tolerance(prec):
    """120x60x30 (config c2): bitwise via the reference's sha256, fast within tol."""
    h = load_golden("hashes.json")
    m, edof, bcs, rho, v = seeded_case((120, 60, 30), 42)
    ex = _op(m, edof, bcs, rho, prec, exact=True)
    got = ex.apply(v.astype(ex.precision.dtype))
    assert _sha(got) == h[f"apply_fused_{prec}_120x60x30"]["sha256"]
    for kernel in ("tile", "pull"):
        fast = _op(m, edof, bcs, rho, prec, grid_kernel=kernel)
        w = fast.apply(v.astype(fast.precision.dtype))
        assert _rel(w, got) <= TOL[prec], kernel


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_diagonal_bitwise(prec):
    for dims, seed in SMALL[:2]:
        g = load_golden(f"matvec_{'x'.join(map(str, dims))}.npz")
        m, edof, bcs, rho, v = seeded_case(dims, seed)
        op = _op(m, edof, bcs, rho, prec)
        assert np.array_equal(op.diagonal(), g[f"diag_{prec}"])


def test_energies_match_reference():
    for dims, seed in SMALL:
        g = load_golden(f"matvec_{'x'.join(map(str, dims))}.npz")
        m, edof, bcs, rho, v = seeded_case(dims, seed)
        op = _op(m, edof, bcs, rho, "fp64")
        assert _rel(op.element_energies(v), g["energies"]) <= 1e-12


def test_energies_ignore_rigid_translation():
    """A deformation d carried along by a huge rigid translation: the parity-
    basis energy drops the translation before any product, so E(d + t) equals
    E(d) to round-off of the deformation (the direct u^T Ke u form would carry
    eps*|Ke|*|t|^2 ~ 1e0 here and can go negative)."""
    import oracle

    m, edof, bcs, rho, v = seeded_case((6, 5, 4), 7)
    op = _op(m, edof, bcs, rho, "fp64")
    t = np.tile([3e8, -1e8, 2e8], m.n_nodes)
    e_d = op.element_energies(v)
    e_u = op.element_energies(v + t)
    assert np.abs(e_u - e_d).max() <= 1e-5 * np.abs(e_d).max()
    assert e_u.min() >= 0.0
    # the reference's direct form on the same input (the checker): noise of ~|t|^2 eps
    e_ref = oracle.element_energies(edof, op.ke64, v + t)
    assert np.abs(e_ref - e_d).max() > 1e-3 * np.abs(e_d).max()


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
@pytest.mark.parametrize("scatter", ["serial", "parallel_atomic"])
def test_general_edof_kernels_seeded_random(prec, scatter):
    """Non-structured connectivity (the bench's seeded_random DOF relabel)."""
    from paper_2604_18020_b200 import BoundaryConditions

    m, edof, bcs, rho, v = seeded_case((16, 8, 4), 42)
    rng = np.random.default_rng(5)
    perm = rng.permutation(m.n_dof).astype(np.int32)
    edof_p = np.ascontiguousarray(perm[edof])
    bcs_p = BoundaryConditions(np.sort(perm[bcs.fixed_dofs]), np.zeros(m.n_dof))
    op = _op(m, edof_p, bcs_p, rho, prec, scatter=scatter)
    assert not op.structured
    got = op.apply(v.astype(op.precision.dtype))
    want = oracle.apply(edof_p, op.ke, op.scale, v, bcs_p.fixed_dofs, m.n_dof)
    assert _rel(got, want) <= TOL[prec]
    if scatter == "serial":  # the reference's element order: bitwise fused_serial
        assert np.array_equal(got, want)
        for _ in range(3):
            assert np.array_equal(op.apply(v.astype(op.precision.dtype)), got)


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_three_stage_variant(prec):
    g = load_golden("matvec_24x12x6.npz")
    m, edof, bcs, rho, v = seeded_case((24, 12, 6), 42)
    op = _op(m, edof, bcs, rho, prec, variant="three_stage")
    assert _rel(op.apply(v.astype(op.precision.dtype)), g[f"apply_three_stage_{prec}"]) <= TOL[prec]


def test_fixed_pass_through_and_masking():
    m, edof, bcs, rho, v = seeded_case((6, 4, 3), 3)
    op = _op(m, edof, bcs, rho, "fp64")
    w = op.apply(v)
    assert np.array_equal(w[bcs.fixed_dofs], v[bcs.fixed_dofs])
    v2 = v.copy()
    v2[bcs.fixed_dofs] += 1.0
    w2 = op.apply(v2)
    free = bcs.free_mask(m.n_dof)
    assert np.array_equal(w2[free], w[free])


def test_repeated_apply_bitwise_stable():
    m, edof, bcs, rho, v = seeded_case((40, 20, 10), 9)
    for prec in ("fp64", "fp32"):
        op = _op(m, edof, bcs, rho, prec)
        first = op.apply(v.astype(op.precision.dtype))
        for _ in range(5):
            assert np.array_equal(op.apply(v.astype(op.precision.dtype)), first)


def test_large_properties_symmetry_linearity():
    """Size-independent properties at c4 size (1M elements)."""
    import torch

    from paper_2604_18020_b200 import make_preset

    pb = make_preset("cantilever", 5 / 3)
    m = pb.mesh
    rng = np.random.default_rng(1)
    rho = rng.uniform(0.05, 1.0, m.n_elem)
    from paper_2604_18020_b200 import build_edof

    op = _op(m, build_edof(m), pb.bcs, rho, "fp64")
    x = torch.tensor(rng.standard_normal(m.n_dof), device="cuda")
    y = torch.tensor(rng.standard_normal(m.n_dof), device="cuda")
    free = torch.tensor(pb.bcs.free_mask(m.n_dof), device="cuda")
    x = x * free
    y = y * free
    kx, ky = op.apply(x), op.apply(y)
    a, b = float(torch.dot(y, kx)), float(torch.dot(x, ky))
    assert abs(a - b) <= 1e-12 * abs(a) * 10
    k2 = op.apply(2.0 * x + 3.0 * y)
    assert float((k2 - (2.0 * kx + 3.0 * ky)).abs().max()) <= 1e-12 * float(kx.abs().max()) * 10
    assert float(torch.dot(x, kx)) > 0.0


@pytest.mark.parametrize("dims", [(1, 1, 1), (2, 1, 1), (31, 7, 3), (32, 8, 17), (63, 15, 40),
                                  (7, 50, 9), (100, 3, 2)])
@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_tile_kernel_edge_shapes(dims, prec):
    """Tile/chunk boundaries (31x7 node columns per CTA, z chunks) vs the oracle."""
    m, edof, bcs, rho, v = seeded_case(dims, 77)
    op = _op(m, edof, bcs, rho, prec)
    got = op.apply(v.astype(op.precision.dtype))
    want = oracle.apply(edof, op.ke, op.scale, v, bcs.fixed_dofs, m.n_dof)
    assert _rel(got, want) <= TOL[prec]


def test_tile_falls_back_for_unstructured_ke():
    """A Ke without the mirror-parity block structure must use the dense kernel."""
    m, edof, bcs, rho, v = seeded_case((6, 5, 4), 3)
    op = _op(m, edof, bcs, rho, "fp64")
    rng = np.random.default_rng(0)
    a = rng.standard_normal((24, 24))
    op.ke = np.ascontiguousarray(a + a.T)
    got = op.apply(v)
    want = oracle.apply(edof, op.ke, op.scale, v, bcs.fixed_dofs, m.n_dof)
    assert _rel(got, want) <= 1e-12


def test_apply_stream_matches_apply():
    """Pipelined host-to-host applies (the e2e path) equal one-by-one applies."""
    import torch

    m, edof, bcs, rho, v = seeded_case((30, 12, 10), 21)
    op = _op(m, edof, bcs, rho, "fp32")
    rng = np.random.default_rng(3)
    vs = [torch.from_numpy(rng.standard_normal(m.n_dof).astype(np.float32)).pin_memory() for _ in range(5)]
    ws = [torch.empty_like(vs[0]).pin_memory() for _ in range(5)]
    op.apply_stream(vs, ws)
    torch.cuda.synchronize()
    for a, b in zip(vs, ws):
        assert np.array_equal(b.numpy(), op.apply(a.numpy()))
    # fp64, odd batch, and a Ke without the parity structure (Python pipeline)
    op64 = _op(m, edof, bcs, rho, "fp64")
    vs64 = [torch.from_numpy(rng.standard_normal(m.n_dof)).pin_memory() for _ in range(3)]
    ws64 = [torch.empty_like(vs64[0]).pin_memory() for _ in range(3)]
    op64.apply_stream(vs64, ws64)
    torch.cuda.synchronize()
    for a, b in zip(vs64, ws64):
        assert np.array_equal(b.numpy(), op64.apply(a.numpy()))
    a_ = rng.standard_normal((24, 24))
    op64.ke = np.ascontiguousarray(a_ + a_.T)
    op64.apply_stream(vs64, ws64)
    torch.cuda.synchronize()
    for a, b in zip(vs64, ws64):
        assert np.array_equal(b.numpy(), op64.apply(a.numpy()))


@pytest.mark.parametrize("preset", ["mbb", "bridge", "torsion", "cantilever"])
@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_presets_matvec_and_diagonal_vs_oracle(preset, prec):
    """Every preset's constraint pattern (z-varying pins: mbb; edge rollers:
    bridge; clamped faces) through the structured kernels vs the oracle."""
    from paper_2604_18020_b200 import make_preset

    pb = make_preset(preset, 0.2)
    m = pb.mesh
    from paper_2604_18020_b200 import build_edof

    edof = build_edof(m)
    rng = np.random.default_rng(8)
    rho = rng.uniform(0.05, 1.0, m.n_elem)
    v = rng.standard_normal(m.n_dof)
    for kernel in ("tile", "pull"):
        op = _op(m, edof, pb.bcs, rho, prec, grid_kernel=kernel)
        got = op.apply(v.astype(op.precision.dtype))
        want = oracle.apply(edof, op.ke, op.scale, v, pb.bcs.fixed_dofs, m.n_dof)
        assert _rel(got, want) <= TOL[prec], kernel
    d = op.diagonal()
    assert np.array_equal(d, oracle.diagonal(edof, op.ke, op.scale, pb.bcs.fixed_dofs, m.n_dof))


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_random_constraint_sets_mask_and_pass_through(prec):
    """Arbitrary fixed DOFs (z-varying columns, interior nodes, single
    components) exercise the per-node mask path of the tile kernel."""
    from paper_2604_18020_b200 import BoundaryConditions

    m, edof, bcs, rho, v = seeded_case((40, 9, 13), 5)
    rng = np.random.default_rng(6)
    fixed = np.unique(rng.choice(m.n_dof, size=m.n_dof // 7, replace=False))
    b2 = BoundaryConditions(fixed, np.zeros(m.n_dof))
    op = _op(m, edof, b2, rho, prec)
    got = op.apply(v.astype(op.precision.dtype))
    want = oracle.apply(edof, op.ke, op.scale, v, b2.fixed_dofs, m.n_dof)
    assert _rel(got, want) <= TOL[prec]
    assert np.array_equal(got[fixed], v.astype(op.precision.dtype)[fixed])


def test_no_constraints_rigid_modes_in_null_space():
    """Without supports K annihilates rigid translations (interior rows)."""
    from paper_2604_18020_b200 import BoundaryConditions

    m, edof, bcs, rho, v = seeded_case((17, 11, 9), 2)
    free = BoundaryConditions(np.zeros(0, dtype=np.int64), np.zeros(m.n_dof))
    op = _op(m, edof, free, rho, "fp64")
    for axis in range(3):
        t = np.zeros(m.n_dof)
        t[axis::3] = 1.0
        assert np.abs(op.apply(t)).max() <= 1e-13


def test_accumulate_flag_and_edof_contract_module():
    """The reference kernel-module contract (kernels.py) accumulates into out."""
    from paper_2604_18020_b200 import kernels

    m, edof, bcs, rho, v = seeded_case((6, 4, 3), 4)
    from paper_2604_18020_b200.element import simp_scale, unit_stiffness

    ke = unit_stiffness(0.3)
    scale = simp_scale(rho)
    out = np.ones(m.n_dof)
    kernels.fused_atomic(edof, ke, scale, v, out)
    want = np.ones(m.n_dof)
    oracle.fused_serial(edof, ke, scale, v, want)
    assert _rel(out, want) <= 1e-12
    out2 = np.ones(m.n_dof)
    kernels.fused_serial(edof, ke, scale, v, out2)
    assert np.array_equal(out2, want)  # bitwise _kernels_numba.py:146-162, accumulating
    out3 = np.ones(m.n_dof, dtype=np.float32)
    kernels.fused_serial(edof, ke.astype(np.float32), scale.astype(np.float32), v.astype(np.float32), out3)
    want3 = np.ones(m.n_dof, dtype=np.float32)
    oracle.fused_serial(edof, ke.astype(np.float32), scale.astype(np.float32), v.astype(np.float32), want3)
    assert np.array_equal(out3, want3)
    acc = np.zeros(m.n_dof)
    kernels.jacobi_diag(edof, np.diag(ke).copy(), scale, acc)
    acc_ref = np.zeros(m.n_dof)
    oracle.jacobi_diag(edof, np.diag(ke).copy(), scale, acc_ref)
    assert _rel(acc, acc_ref) <= 1e-14
    u = kernels.gather(edof, v)
    assert np.array_equal(u, oracle.gather(edof, v))
    assert _rel(kernels.element_energies(edof, ke, v), oracle.element_energies(edof, ke, v)) <= 1e-12


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_node_range_launches_compose_bitwise(prec):
    """Interface/interior split used by the x-slab overlap: the union of range
    launches equals the full structured matvec bit for bit."""
    import torch

    from paper_2604_18020_b200 import _device as D
    from paper_2604_18020_b200 import _lib
    from paper_2604_18020_b200.operator import ctypes_ref

    m, edof, bcs, rho, v = seeded_case((90, 13, 11), 31)
    op = _op(m, edof, bcs, rho, prec)
    dt = op.precision.dtype
    x = torch.tensor(v.astype(dt), device="cuda")
    full = op.apply(x)
    out = torch.full_like(x, float("nan"))
    sfx = "f64" if prec == "fp64" else "f32"
    nnx = m.nelx + 1
    for lo, hi in ((0, 31), (nnx - 31, nnx), (31, nnx - 31)):
        _lib.call(f"tf_matvec_grid_range_{sfx}", ctypes_ref(op.dev.grid), op.ke.ctypes.data,
                  D.ptr(op._scale_dev), D.ptr(x), D.ptr(out), D.ptr(op.dev.node_fixed),
                  _lib.TF_MASK_INPUT | _lib.TF_PASS_FIXED, lo, hi, D.stream_ptr())
    assert torch.equal(out, full)


@pytest.mark.parametrize("preset,scale", [("cantilever", 0.2), ("mbb", 0.2), ("bridge", 0.2),
                                          ("torsion", 0.2), ("cantilever", 1.0)])
@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_tile_block_forms_agree(preset, scale, prec, monkeypatch):
    """The tile kernel's two element-block forms -- the generic parity blocks
    (the FP32 CG kernels) and the isotropic form (33 FP ops, scale folded into
    the coefficients; FP64 and FP32 plain products; TF_TILE_GENERIC=1 forces
    the generic form) -- are the same algebra in a different rounding order:
    they agree to round-off, including masked input with z-varying
    constraints (mbb) and pass-through; repeated launches are bitwise equal."""
    import torch

    from paper_2604_18020_b200 import build_edof, make_preset

    pb = make_preset(preset, scale)
    m = pb.mesh
    rng = np.random.default_rng(9)
    rho = rng.uniform(0.05, 1.0, m.n_elem)
    op = _op(m, build_edof(m), pb.bcs, rho, prec)
    v = torch.tensor(rng.standard_normal(m.n_dof), device="cuda").to(
        torch.float64 if prec == "fp64" else torch.float32)
    monkeypatch.setenv("TF_TILE_GENERIC", "1")
    gen = op.apply(v).clone()
    assert torch.equal(op.apply(v), gen)
    monkeypatch.setenv("TF_TILE_GENERIC", "0")
    prod = op.apply(v)  # the isotropic form (every FP64 product, FP32 plain products)
    tol = 1e-13 if prec == "fp64" else 2e-6
    assert float((prod - gen).abs().max()) <= tol * float(gen.abs().max())


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_tile_result_independent_of_z_chunking(prec, monkeypatch):
    """Every DOF is summed in the same order whatever the z-chunk height (the
    chunk's first layer is recomputed, not exchanged), so the autotuned launch
    shape cannot change results: bitwise equal across heights."""
    import torch

    from paper_2604_18020_b200 import build_edof, make_preset

    pb = make_preset("mbb", 0.2)
    m = pb.mesh
    rng = np.random.default_rng(4)
    op = _op(m, build_edof(m), pb.bcs, rng.uniform(0.05, 1.0, m.n_elem), prec)
    v = torch.tensor(rng.standard_normal(m.n_dof), device="cuda").to(
        torch.float64 if prec == "fp64" else torch.float32)
    outs = []
    for oz in ("2", "3", "5", "16"):
        monkeypatch.setenv("TF_TILE_OZ", oz)
        outs.append(op.apply(v).clone())
    for o in outs[1:]:
        assert torch.equal(outs[0], o)


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
@pytest.mark.parametrize("relabel", [False, True])
def test_merged_atomic_edof_matches_oracle(prec, relabel, monkeypatch):
    """The production general-edof atomic product (tf_matvec_edof_merged_*:
    precomputed neighbour-merge mask, constrained slots scattered onto their
    own DOF and overwritten by the pass-through) against the oracle and the
    v2 kernel, on the structured numbering and a seeded DOF relabel, with a
    partial last block."""
    import torch

    from paper_2604_18020_b200 import BoundaryConditions

    m, edof, bcs, rho, v = seeded_case((13, 7, 5), 8)  # 455 elements: 3 full blocks + 71
    if relabel:
        perm = np.random.default_rng(2).permutation(m.n_dof).astype(np.int32)
        edof = np.ascontiguousarray(perm[edof])
        bcs = BoundaryConditions(np.sort(perm[bcs.fixed_dofs]), np.zeros(m.n_dof))
    op = _op(m, edof, bcs, rho, prec, grid_kernel="edof", scatter="parallel_atomic")
    assert not op.structured
    got = op.apply(v.astype(op.precision.dtype))
    want = oracle.apply(edof, op.ke, op.scale, v, bcs.fixed_dofs, m.n_dof)
    assert _rel(got, want) <= TOL[prec]
    assert np.array_equal(got[bcs.fixed_dofs], v.astype(op.precision.dtype)[bcs.fixed_dofs])
    monkeypatch.setenv("TF_EDOF_MERGED", "0")
    v2 = op.apply(v.astype(op.precision.dtype))
    assert _rel(v2, got) <= TOL[prec]
    # x-neighbours inside a warp and a mesh row share a face: 12 pairs (a
    # DOF relabel keeps which slots coincide, so the mask is the same)
    mask = op.dev.merge_mask().cpu().numpy().astype(np.uint16)
    lanes = np.arange(m.n_elem) % 32
    ex = np.arange(m.n_elem) % m.nelx
    inner = (lanes != 31) & (ex != m.nelx - 1)
    assert np.all(mask[inner] == 0xFFF)
    assert np.all(mask[~inner] == 0)


def test_merge_mask_rejects_minus_one_slots():
    """The merged atomic product adds a masked slot's row to the DOF in its low
    31 bits, so the connectivity check refuses -1 slots (which would address
    DOF 2^31-1) instead of letting a product write out of bounds."""
    import torch

    from paper_2604_18020_b200 import _device as D
    from paper_2604_18020_b200 import _lib

    m, edof, bcs, rho, v = seeded_case((4, 3, 2), 11)
    bad = edof.astype(np.int32).copy()
    bad[0, 5] = -1
    e_d = torch.tensor(bad, device="cuda")
    mask = torch.empty(m.n_elem, dtype=torch.int16, device="cuda")
    with pytest.raises(_lib.TfError, match="low 31 bits"):
        _lib.call("tf_edof_merge_mask", D.ptr(e_d), m.n_elem, m.n_dof, D.ptr(mask), D.stream_ptr())
    good = torch.tensor(D.masked_edof(edof, bcs.fixed_dofs, m.n_dof), device="cuda")
    _lib.call("tf_edof_merge_mask", D.ptr(good), m.n_elem, m.n_dof, D.ptr(mask), D.stream_ptr())
