"""Unit-cube trilinear hex stiffness and SIMP material interpolation.

Mirrors reference ``topofuse.element`` (element.py:20-135).  The 24x24
``unit_stiffness`` is built here from the closed-form integrals of products of
trilinear shape-function gradients over the unit cube (exact, no quadrature
loop), then symmetrised; it agrees with the reference's 2x2x2 Gauss build to
round-off (tests/test_host.py pins it against the reference bitwise-golden at
1e-14, the reference's own tolerance, test_element.py:20-24).

For an isotropic material, K_ab[c][d] = lam*I_cd + mu*(delta_cd*sum_p I_pp + I_dc)
with I_pq = int dN_a/dx_p dN_b/dx_q dV; on the unit cube every I_pq factorises
into per-axis 1-D integrals of (1 + s t) factors.
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from .mesh import CORNER_OFFSETS, StructuredMesh

RHO_MIN = 1e-9
DENSE_DOF_LIMIT = 10_000


@dataclass(frozen=True)
class SimpParams:
    """E(rho) = rho_min + (1 - rho_min) * rho**p (reference element.py:20-31)."""

    p: float = 3.0
    rho_min: float = RHO_MIN

    def __post_init__(self):
        if self.p < 1.0:
            raise ValueError("penalization exponent must be >= 1")
        if not (0.0 < self.rho_min < 1.0):
            raise ValueError("rho_min must lie in (0, 1)")


def simp_scale(rho, params: SimpParams = SimpParams()):
    """Per-element stiffness factor (reference element.py:34-39)."""
    rho = np.asarray(rho)
    if rho.size and (rho.min() < -1e-12 or rho.max() > 1.0 + 1e-12):
        raise ValueError("densities must lie in [0, 1]")
    return params.rho_min + (1.0 - params.rho_min) * np.clip(rho, 0.0, 1.0) ** params.p


def simp_scale_derivative(rho, params: SimpParams = SimpParams()):
    """d simp_scale / d rho (reference element.py:42-45)."""
    r = np.clip(np.asarray(rho), 0.0, 1.0)
    return params.p * (1.0 - params.rho_min) * r ** (params.p - 1.0)


def elasticity_matrix(nu: float) -> np.ndarray:
    """Voigt (xx, yy, zz, yz, xz, xy) isotropic stiffness, E = 1."""
    lam = nu / ((1.0 + nu) * (1.0 - 2.0 * nu))
    mu = 0.5 / (1.0 + nu)
    d = np.zeros((6, 6))
    d[:3, :3] = lam
    d[[0, 1, 2], [0, 1, 2]] = lam + 2.0 * mu
    d[[3, 4, 5], [3, 4, 5]] = mu
    return d


def _gradient_integrals() -> np.ndarray:
    """I[a, b, p, q] = int_{[0,1]^3} dN_a/dx_p * dN_b/dx_q dV for the 8 corners."""
    s = 2.0 * CORNER_OFFSETS - 1.0  # corner signs in [-1, 1]^3
    # 1-D integrals over t in [-1, 1] with the 1/2 Jacobian per axis folded in:
    # int (1 + a t)(1 + b t) dt = 2 + 2ab/3 ; int (1 + a t) dt = 2 ; int dt = 2
    I = np.zeros((8, 8, 3, 3))
    for a in range(8):
        for b in range(8):
            pair = 2.0 + (2.0 / 3.0) * s[a] * s[b]  # per-axis value-value integral
            for p in range(3):
                for q in range(3):
                    if p == q:
                        val = s[a, p] * s[b, p] * 2.0
                        for r in range(3):
                            if r != p:
                                val *= pair[r]
                    else:
                        r = 3 - p - q
                        val = s[a, p] * s[b, q] * 2.0 * 2.0 * pair[r]
                    # dN/dx = 2 dN/dxi -> (1/4 s ...) each; dV = dxi/8
                    I[a, b, p, q] = val / 16.0 / 8.0
    return I


@lru_cache(maxsize=8)
def unit_stiffness(nu: float = 0.3) -> np.ndarray:
    """24x24 stiffness of the unit-cube element, E = 1 (read-only, cached)."""
    lam = nu / ((1.0 + nu) * (1.0 - 2.0 * nu))
    mu = 0.5 / (1.0 + nu)
    I = _gradient_integrals()
    trace = I[:, :, 0, 0] + I[:, :, 1, 1] + I[:, :, 2, 2]
    k = np.zeros((8, 3, 8, 3))
    for c in range(3):
        for d in range(3):
            blk = lam * I[:, :, c, d] + mu * I[:, :, d, c]
            if c == d:
                blk = blk + mu * trace
            k[:, c, :, d] = blk
    ke = k.reshape(24, 24)
    ke = 0.5 * (ke + ke.T)
    ke.setflags(write=False)
    return ke


def assemble_dense(mesh: StructuredMesh, edof: np.ndarray, scaled_density: np.ndarray,
                   fixed_dofs=None, nu: float = 0.3) -> np.ndarray:
    """Dense K for verification meshes only (reference element.py:106-135)."""
    if mesh.n_dof > DENSE_DOF_LIMIT:
        raise ValueError(f"dense assembly limited to {DENSE_DOF_LIMIT} DOFs, mesh has {mesh.n_dof}")
    ke = unit_stiffness(nu)
    k = np.zeros((mesh.n_dof, mesh.n_dof))
    edof = np.asarray(edof, dtype=np.int64)
    for e in range(edof.shape[0]):
        idx = edof[e]
        k[idx[:, None], idx[None, :]] += scaled_density[e] * ke
    if fixed_dofs is not None and len(fixed_dofs):
        f = np.asarray(fixed_dofs, dtype=np.int64)
        k[f, :] = 0.0
        k[:, f] = 0.0
        k[f, f] = 1.0
    return k
