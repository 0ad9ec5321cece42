"""Pin the CPU oracle against outputs of the real reference (golden fixtures).

The oracle (oracle/) is the checker for every GPU parity test, so it must
itself reproduce the reference bitwise: FP64 and FP32 (numba order) fused
serial, three-stage, Jacobi diagonal and element energies, and the full-size
sha256 hashes recorded from the reference at 48x24x24 and 120x60x30.
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

import oracle
from conftest import load_golden, seeded_case
from paper_2604_18020_b200.element import SimpParams, simp_scale

SMALL = [((4, 3, 2), 11), ((5, 3, 2), 12), ((1, 1, 1), 1001), ((24, 12, 6), 42)]


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _ops(golden_ke, rho, prec):
    dt = np.float64 if prec == "fp64" else np.float32
    scale = np.asarray(simp_scale(rho, SimpParams(3.0)), dtype=np.float64).astype(dt)
    return np.ascontiguousarray(golden_ke, dtype=dt), scale, dt


@pytest.mark.parametrize("dims,seed", SMALL)
@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_oracle_apply_bitwise_vs_reference(golden_ke, dims, seed, prec):
    g = load_golden(f"matvec_{'x'.join(map(str, dims))}.npz")
    m, edof, bcs, rho, v = seeded_case(dims, seed)
    ke, scale, dt = _ops(golden_ke, rho, prec)
    for variant in ("fused", "three_stage"):
        got = oracle.apply(edof, ke, scale, v, bcs.fixed_dofs, m.n_dof, variant)
        want = g[f"apply_{variant}_{prec}"]
        assert got.dtype == want.dtype
        assert np.array_equal(got, want), (variant, np.abs(got - want).max())
    out = np.zeros(m.n_dof, dtype=dt)
    oracle.fused_serial(edof, ke, scale, v.astype(dt), out)
    assert np.array_equal(out, g[f"raw_fused_{prec}"])
    d = oracle.diagonal(edof, ke, scale, bcs.fixed_dofs, m.n_dof)
    assert np.array_equal(d, g[f"diag_{prec}"])


@pytest.mark.parametrize("dims,seed", SMALL)
def test_oracle_energies_bitwise(golden_ke, dims, seed):
    g = load_golden(f"matvec_{'x'.join(map(str, dims))}.npz")
    m, edof, bcs, rho, v = seeded_case(dims, seed)
    assert np.array_equal(oracle.element_energies(edof, golden_ke, v), g["energies"])


@pytest.mark.parametrize("dims", [(48, 24, 24), (120, 60, 30)])
def test_oracle_full_size_hashes(golden_ke, dims):
    """Bitwise at BASELINE sizes (c1 and c2) via the reference's sha256."""
    h = load_golden("hashes.json")
    tag = "x".join(map(str, dims))
    m, edof, bcs, rho, v = seeded_case(dims, 42)
    assert _sha(edof) == h[f"edof_{tag}"]
    for prec in ("fp64", "fp32"):
        ke, scale, dt = _ops(golden_ke, rho, prec)
        got = oracle.apply(edof, ke, scale, v, bcs.fixed_dofs, m.n_dof, "fused")
        assert _sha(got) == h[f"apply_fused_{prec}_{tag}"]["sha256"], prec
        d = oracle.diagonal(edof, ke, scale, bcs.fixed_dofs, m.n_dof)
        assert _sha(d) == h[f"diag_{prec}_{tag}"]["sha256"], prec
    assert _sha(oracle.element_energies(edof, golden_ke, v)) == h[f"energies_{tag}"]["sha256"]


def test_oracle_atomic_matches_serial_within_tolerance(golden_ke):
    m, edof, bcs, rho, v = seeded_case((24, 12, 6), 42)
    for prec, tol in (("fp64", 1e-12), ("fp32", 1e-5)):
        ke, scale, dt = _ops(golden_ke, rho, prec)
        a = np.zeros(m.n_dof, dt)
        b = np.zeros(m.n_dof, dt)
        oracle.fused_serial(edof, ke, scale, v.astype(dt), a)
        oracle.fused_atomic(edof, ke, scale, v.astype(dt), b, threads=4)
        assert np.abs(a - b).max() <= tol * np.abs(a).max()


def test_oracle_pcg_matches_reference_anchor(golden_ke):
    """Cold solve on the desk cantilever: iteration count and history."""
    from paper_2604_18020_b200.mesh import build_edof, make_preset

    cg = load_golden("cg.json")["desk_fp64"]
    pb = make_preset("cantilever", 0.2)
    m = pb.mesh
    edof = build_edof(m)
    ke, scale, dt = _ops(golden_ke, np.full(m.n_elem, 0.5), "fp64")
    A = lambda x: oracle.apply(edof, ke, scale, x, pb.bcs.fixed_dofs, m.n_dof)
    diag = oracle.diagonal(edof, ke, scale, pb.bcs.fixed_dofs, m.n_dof)
    x, info = oracle.pcg(A, pb.bcs.force.copy(), diag)
    assert info["iterations"] == cg["iterations"]
    np.testing.assert_allclose(info["history"], cg["history"], rtol=1e-9)


# -- emulated BF16 (tests/golden/make_golden_bf16.py) ---------------------------

BF16_CASES = [((4, 3, 2), 11), ((5, 3, 2), 1030)]


def test_oracle_round_bf16_bitwise_vs_reference():
    g = load_golden("bf16_4x3x2.npz")
    got = oracle.round_bf16(g["specials"])
    assert np.array_equal(got.view(np.uint32), g["round_specials"].view(np.uint32))


@pytest.mark.parametrize("dims,seed", BF16_CASES)
def test_oracle_bf16_kernels_bitwise_vs_reference(golden_ke, dims, seed):
    g = load_golden(f"bf16_{'x'.join(map(str, dims))}.npz")
    m, edof, bcs, rho, v = seeded_case(dims, seed)
    ke, scale, _ = _ops(golden_ke, rho, "fp32")
    vq = oracle.round_bf16(v.astype(np.float32))
    out = np.zeros(m.n_dof, dtype=np.float32)
    oracle.fused_serial_bf16(edof, ke, scale, vq, out)
    assert np.array_equal(out, g["raw_fused_serial_bf16"])
    assert np.array_equal(oracle.gemm_bf16(oracle.gather(edof, vq), ke, scale), g["raw_gemm_bf16"])
    d = np.zeros(m.n_dof, dtype=np.float32)
    oracle.jacobi_diag_bf16(edof, np.diag(ke).copy(), scale, d)
    assert np.array_equal(d, g["raw_jacobi_bf16"])
    for variant in ("fused", "three_stage"):
        got = oracle.apply_bf16(edof, ke, scale, v, bcs.fixed_dofs, m.n_dof, variant)
        assert np.array_equal(got, g[f"apply_{variant}"]), variant
    assert np.array_equal(oracle.diagonal_bf16(edof, ke, scale, bcs.fixed_dofs, m.n_dof), g["diag"])


@pytest.mark.parametrize("name", ["c3", "c4", "c5"])
def test_oracle_baseline_size_hashes(golden_ke, name):
    """Bitwise at the remaining BASELINE sizes the bench times (c3 torsion,
    c4 1M, c5 4.9M) via the reference's sha256 (make_golden_r2.py)."""
    from conftest import baseline_case

    h = load_golden("hashes_r2.json")
    m, edof, bcs, rho, v = baseline_case(name)
    for prec in ("fp64", "fp32"):
        ke, scale, dt = _ops(golden_ke, rho, prec)
        got = oracle.apply(edof, ke, scale, v, bcs.fixed_dofs, m.n_dof, "fused")
        assert _sha(got) == h[f"apply_fused_{prec}_{name}"]["sha256"], prec


def test_oracle_simp_restatement_pinned_to_reference_c1():
    """oracle/simp.py (the CPU baseline's SIMP loop) against the reference's
    own c1 trajectory: the first 3 iterations' compliances to 1e-12 and CG
    counts exactly (FP64 serial)."""
    from oracle import simp as osimp
    from paper_2604_18020_b200.element import unit_stiffness
    from paper_2604_18020_b200.mesh import StructuredMesh, build_edof, cantilever_bcs

    g = load_golden("simp_c1_fp64.npz")
    m = StructuredMesh(48, 24, 24)
    b = cantilever_bcs(m)
    hist, _ = osimp.run_simp((48, 24, 24), build_edof(m), b.fixed_dofs, b.force, 0.3,
                             [(1, 30, 3.0, 1.0, 0.2, 1.5)], 1.5, unit_stiffness(0.3), iterations=3)
    c = np.array([r["compliance"] for r in hist])
    np.testing.assert_allclose(c, g["compliance"][:3], rtol=1e-12)
    assert [r["cg_iterations"] for r in hist] == list(g["cg_iterations"][:3])
