"""Emulated-BF16 path on the B200 (csrc/tf_bf16.cu) against the reference.

BF16 is the documented negative result of the north star,
not a production path; these tests pin that the B200 build reproduces the
reference's BF16 contract (precision.py, _kernels_numba.py bf16 kernels,
operator.py bf16 branches, solver.py quantized rules) on the goldens of
tests/golden/make_golden_bf16.py.

Bars: the deterministic (colour-ordered) kernels are bitwise; atomics and the
three-stage gather/GEMM/scatter follow the reference arithmetic per term, with
only the FP32 summation order across elements free (1e-6 of max|w|).
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle
from conftest import load_golden, seeded_case

pytestmark = pytest.mark.gpu

CASES = [((4, 3, 2), 11), ((5, 3, 2), 1030)]


def _op(m, edof, bcs, rho, variant="fused", scatter="serial"):
    from paper_2604_18020_b200 import MatFreeOperator, SimpParams

    return MatFreeOperator(m, edof, bcs, rho, SimpParams(3.0), "bf16", variant, scatter)


@pytest.mark.parametrize("dims,seed", CASES)
def test_bf16_operator_matches_reference(dims, seed):
    g = load_golden(f"bf16_{'x'.join(map(str, dims))}.npz")
    m, edof, bcs, rho, v = seeded_case(dims, seed)
    op = _op(m, edof, bcs, rho)
    assert not op.structured
    v32 = v.astype(np.float32)
    # colour-ordered fused: each DOF sums its elements' rows in colour order,
    # the reference in element order -> FP32 rounding of that sum only
    got = op.apply(v32)
    ref = g["apply_fused"]
    assert np.abs(got - ref).max() <= 1e-6 * np.abs(ref).max()
    for variant, scatter in (("fused", "parallel_atomic"), ("three_stage", "serial")):
        o = _op(m, edof, bcs, rho, variant, scatter)
        ref = g[f"apply_{variant}"]
        assert np.abs(o.apply(v32) - ref).max() <= 1e-6 * np.abs(ref).max()
    d = op.diagonal()
    assert np.abs(d - g["diag"]).max() <= 1e-6 * np.abs(g["diag"]).max()
    a64 = op.apply_fp64(v)
    assert np.abs(a64 - g["apply_fp64"]).max() <= 1e-12 * np.abs(g["apply_fp64"]).max()
    # the fixed-DOF pass-through returns the raw input, unquantized
    assert np.array_equal(got[bcs.fixed_dofs], v32[bcs.fixed_dofs])


@pytest.mark.parametrize("dims,seed", CASES)
def test_bf16_contract_kernels_match_reference(dims, seed):
    from paper_2604_18020_b200 import kernels as K

    g = load_golden(f"bf16_{'x'.join(map(str, dims))}.npz")
    m, edof, bcs, rho, v = seeded_case(dims, seed)
    op = _op(m, edof, bcs, rho)
    vq = oracle.round_bf16(v.astype(np.float32))
    for fn in (K.fused_serial_bf16, K.fused_atomic_bf16):
        out = np.zeros(m.n_dof, dtype=np.float32)
        fn(edof, op.ke, op.scale, vq, out)
        ref = g["raw_fused_serial_bf16"]
        assert np.abs(out - ref).max() <= 1e-6 * np.abs(ref).max()
    # per element: no cross-element sums -> bitwise
    assert np.array_equal(K.gemm_bf16(oracle.gather(edof, vq), op.ke, op.scale), g["raw_gemm_bf16"])
    d = np.zeros(m.n_dof, dtype=np.float32)
    K.jacobi_diag_bf16(edof, np.diag(op.ke).copy(), op.scale, d)
    assert np.abs(d - g["raw_jacobi_bf16"]).max() <= 1e-6 * np.abs(g["raw_jacobi_bf16"]).max()


def test_bf16_round_is_bitwise():
    import torch

    from paper_2604_18020_b200 import _device as D, _lib

    g = load_golden("bf16_4x3x2.npz")
    x = torch.tensor(g["specials"], device="cuda")
    y = torch.empty_like(x)
    _lib.call("tf_round_bf16", x.numel(), D.ptr(x), D.ptr(y), D.stream_ptr())
    assert np.array_equal(y.cpu().numpy().view(np.uint32), g["round_specials"].view(np.uint32))


def test_bf16_cold_solve_and_refinement_reproduce_the_negative_result():
    """Desk cantilever (reference solver.py rules): the bf16 cold solve stops
    on its recurrence but fails the FP64 verification ('floor') with a wrong
    compliance; iterative refinement does not reach 1e-5 in 8 outer steps."""
    from paper_2604_18020_b200 import (CgConfig, MatFreeOperator, SimpParams, build_edof, make_preset,
                                       solve_equilibrium, solve_refined)

    gs = load_golden("bf16_solve.json")
    pb = make_preset("cantilever", 0.2)
    edof = build_edof(pb.mesh)
    rho = np.full(pb.mesh.n_elem, 0.5)
    op16 = MatFreeOperator(pb.mesh, edof, pb.bcs, rho, SimpParams(3.0), "bf16")
    u, rep = solve_equilibrium(op16, pb.bcs.force, CgConfig())
    g = gs["desk_bf16"]
    assert rep.termination == g["termination"] == "floor"
    assert abs(rep.iterations - g["iterations"]) <= max(2, 0.02 * g["iterations"])
    assert abs(rep.compliance - g["compliance"]) <= 1e-3 * g["compliance"]
    assert abs(rep.verified_rel_residual - g["verified_rel_residual"]) <= 0.05 * g["verified_rel_residual"]
    assert rep.matvecs == rep.iterations  # no true-residual refresh for quantized operators
    op32 = MatFreeOperator(pb.mesh, edof, pb.bcs, rho, SimpParams(3.0), "fp32")
    _, ir = solve_refined(op32, op16, pb.bcs.force)
    gi = gs["desk_ir"]
    assert ir.converged == gi["converged"] and ir.stagnated == gi["stagnated"]
    assert ir.outer_steps == gi["outer_steps"]
    np.testing.assert_allclose(ir.outer_residuals, gi["outer_residuals"], rtol=0.05)
    assert abs(ir.compliance - gi["compliance"]) <= 0.02 * abs(gi["compliance"])


def test_quantize_krylov_rounds_the_recurrence():
    """CgConfig(quantize_krylov=True) on an fp32 operator: the device recurrence
    rounds p and r to bf16 each iteration like the reference's pcg
    (solver.py:134-136); compared with the oracle recurrence with the same rule."""
    from paper_2604_18020_b200 import CgConfig, MatFreeOperator, SimpParams, build_edof, make_preset, pcg

    pb = make_preset("cantilever", 0.2)
    edof = build_edof(pb.mesh)
    rho = np.full(pb.mesh.n_elem, 0.5)
    op = MatFreeOperator(pb.mesh, edof, pb.bcs, rho, SimpParams(3.0), "fp32")
    b = pb.bcs.force.astype(np.float32)
    d = op.diagonal()
    x, rep = pcg(op, b, d, CgConfig(max_iter=30, quantize_krylov=True))
    xr, info = oracle.pcg(lambda z: oracle.apply(edof, op.ke, op.scale, z, pb.bcs.fixed_dofs, pb.mesh.n_dof),
                          b, d, max_iter=30, quantize_krylov=True)
    assert rep.iterations == info["iterations"] == 30
    # bf16-rounded Krylov vectors: agreement to bf16 resolution
    assert np.abs(x - xr).max() <= 2e-2 * np.abs(xr).max()
    with pytest.raises(ValueError):
        op64 = MatFreeOperator(pb.mesh, edof, pb.bcs, rho, SimpParams(3.0), "fp64")
        pcg(op64, pb.bcs.force, op64.diagonal(), CgConfig(quantize_krylov=True))
