"""Unit-cube trilinear hex stiffness and SIMP material interpolation.

Mirrors reference ``topofuse.element`` (element.py:20-135).  The 24x24
``unit_stiffness`` is the reference's 2x2x2 Gauss build with the reference's
roundings, bitwise (tests/test_host.py compares all 576 FP64 entries with the
matrix the reference itself produced), so every kernel that consumes Ke --
the bitwise verification mode, the Jacobi diagonal -- is the reference's
arithmetic through the public API, with no golden matrix injected.
"""

from __future__ import annotations

from dataclasses import dataclass
import itertools
from fractions import Fraction
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
    """Voigt (xx, yy, zz, yz, xz, xy) isotropic stiffness, E = 1, formed with
    the reference's roundings (element.py:59-66): c = 1/((1+nu)(1-2nu)),
    normal block c*nu / c*(1-nu), shear 0.5/(1+nu)."""
    c = 1.0 / ((1.0 + nu) * (1.0 - 2.0 * nu))
    d = np.zeros((6, 6))
    d[:3, :3] = c * nu
    d[[0, 1, 2], [0, 1, 2]] = c * (1.0 - nu)
    d[[3, 4, 5], [3, 4, 5]] = 0.5 / (1.0 + nu)
    return d


# Strain rows (Voigt) fed by each displacement component: (row, component,
# gradient axis) triples of the symmetric gradient.
_STRAIN_PATTERN = ((0, 0, 0), (1, 1, 1), (2, 2, 2), (3, 1, 2), (3, 2, 1),
                   (4, 0, 2), (4, 2, 0), (5, 0, 1), (5, 1, 0))


def _strain_matrix(pt) -> np.ndarray:
    """B (6 x 24) at a reference point of [-1, 1]^3 for the unit cube
    (dN/dx = 2 dN/dxi), gradients rounded as the reference rounds them
    (element.py:47-56: 0.125*s_i, times the two (1 + s t) factors in axis
    order, then the exact factor 2)."""
    s = 2.0 * CORNER_OFFSETS - 1.0
    b = np.zeros((6, 24))
    for a in range(8):
        g = np.empty(3)
        for i in range(3):
            j, k = [ax for ax in range(3) if ax != i]
            g[i] = 0.125 * s[a, i] * (1.0 + s[a, j] * pt[j]) * (1.0 + s[a, k] * pt[k])
        g *= 2.0
        for row, comp, axis in _STRAIN_PATTERN:
            b[row, 3 * a + comp] = g[axis]
    return b


def _fma_chain(t_row: np.ndarray, b_col: np.ndarray) -> float:
    """sum_k t_k b_k as a chain of correctly rounded fused multiply-adds from
    0.0 in ascending k -- the rounding of the OpenBLAS dgemm micro-kernel the
    reference's ``b.T @ d @ b`` reaches (probed against the reference's Ke:
    this chain reproduces all 576 entries bitwise, a plain sum differs in
    161).  Exact rational arithmetic makes it host-independent."""
    acc = Fraction(0)
    out = 0.0
    for tk, bk in zip(t_row.tolist(), b_col.tolist()):
        acc = Fraction(tk) * Fraction(bk) + Fraction(out)
        out = float(acc)  # int/int true division: correctly rounded
    return out


@lru_cache(maxsize=8)
def unit_stiffness(nu: float = 0.3) -> np.ndarray:
    """24x24 stiffness of the unit-cube element, E = 1 (read-only, cached).

    2x2x2 Gauss quadrature with det J = 1/8, accumulated over the points in
    (xi, eta, zeta) nesting order and symmetrised -- the reference's build
    (element.py:69-101), reproduced bitwise: ``tests/test_host.py`` compares
    all 576 FP64 entries with the reference's own matrix (golden ke.npz).
    """
    d = elasticity_matrix(nu)
    g = 1.0 / np.sqrt(3.0)
    ke = np.zeros((24, 24))
    for pt in itertools.product((-g, g), repeat=3):
        b = _strain_matrix(pt)
        t = b.T @ d  # d is block diagonal: each entry is at most 3 exact-order terms
        m = np.empty((24, 24))
        for i in range(24):
            for j in range(24):
                m[i, j] = _fma_chain(t[i], b[:, j])
        ke += m * 0.125
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
