"""Structured hex grids, element->DOF maps, supports and load cases.

Host-side input contract of the hot path, mirroring the reference
``topofuse.mesh`` API (mesh.py:34-246): same names, numbering and presets,
so an existing caller builds identical problems.

Numbering (reference mesh.py:4-7, 58-63): nodes and elements are x-fastest,
node(i, j, k) = i + (nx+1)*(j + (ny+1)*k); node n owns DOFs 3n, 3n+1, 3n+2.
Corner order inside an element (mesh.py:19-31): bottom face counter-clockwise
(000, 100, 110, 010), then the top face in the same order.

B200 note: the device kernels never read the edof table for a structured
grid -- connectivity is index arithmetic on (ex, ey, ez).  ``build_edof`` is
kept for the reference contract and for the general-connectivity kernels.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

# bottom face CCW, then top face CCW  (reference mesh.py:19-31)
CORNER_OFFSETS = np.array(
    [[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0],
     [0, 0, 1], [1, 0, 1], [1, 1, 1], [0, 1, 1]],
    dtype=np.int64,
)


@dataclass(frozen=True)
class StructuredMesh:
    """nelx x nely x nelz unit-cube hexahedra (reference mesh.py:34-80)."""

    nelx: int
    nely: int
    nelz: int

    def __post_init__(self):
        if self.nelx < 1 or self.nely < 1 or self.nelz < 1:
            raise ValueError("element counts must be positive")

    @property
    def n_elem(self) -> int:
        return self.nelx * self.nely * self.nelz

    @property
    def n_nodes(self) -> int:
        return (self.nelx + 1) * (self.nely + 1) * (self.nelz + 1)

    @property
    def n_dof(self) -> int:
        return 3 * self.n_nodes

    @property
    def node_dims(self) -> tuple[int, int, int]:
        return (self.nelx + 1, self.nely + 1, self.nelz + 1)

    def node_id(self, i, j, k):
        nx1, ny1 = self.nelx + 1, self.nely + 1
        return i + nx1 * (j + ny1 * k)

    def element_id(self, ei, ej, ek):
        return ei + self.nelx * (ej + self.nely * ek)

    def node_grid(self) -> np.ndarray:
        """(n_nodes, 3) integer node coordinates in id order."""
        nx1, ny1, nz1 = self.node_dims
        ids = np.arange(self.n_nodes, dtype=np.int64)
        return np.stack([ids % nx1, (ids // nx1) % ny1, ids // (nx1 * ny1)], axis=1)

    def element_centers(self) -> np.ndarray:
        ids = np.arange(self.n_elem, dtype=np.int64)
        nx, ny = self.nelx, self.nely
        return np.stack([ids % nx + 0.5, (ids // nx) % ny + 0.5, ids // (nx * ny) + 0.5], axis=1)


def element_corner_nodes(mesh: StructuredMesh) -> np.ndarray:
    """(n_elem, 8) int64 global node ids of each element's corners."""
    e = np.arange(mesh.n_elem, dtype=np.int64)
    ex = e % mesh.nelx
    ey = (e // mesh.nelx) % mesh.nely
    ez = e // (mesh.nelx * mesh.nely)
    base = mesh.node_id(ex, ey, ez)
    nx1, ny1 = mesh.nelx + 1, mesh.nely + 1
    off = CORNER_OFFSETS[:, 0] + nx1 * (CORNER_OFFSETS[:, 1] + ny1 * CORNER_OFFSETS[:, 2])
    return base[:, None] + off[None, :]


def build_edof(mesh: StructuredMesh) -> np.ndarray:
    """(n_elem, 24) int32 element->DOF table (reference mesh.py:83-102)."""
    nodes = element_corner_nodes(mesh)
    if 3 * int(nodes[-1, 6]) + 2 >= np.iinfo(np.int32).max:
        raise ValueError("mesh too large for int32 DOF indices")
    edof = (3 * nodes)[:, :, None] + np.arange(3, dtype=np.int64)[None, None, :]
    return np.ascontiguousarray(edof.reshape(mesh.n_elem, 24), dtype=np.int32)


def edof_is_structured(mesh: StructuredMesh, edof: np.ndarray) -> bool:
    """True when `edof` is exactly build_edof(mesh) (selects the index-free kernels)."""
    edof = np.asarray(edof)
    if edof.shape != (mesh.n_elem, 24):
        return False
    step = 1 << 18  # compare in slabs of elements to bound host memory
    full = build_edof(StructuredMesh(mesh.nelx, mesh.nely, 1))
    per_layer = 3 * (mesh.nelx + 1) * (mesh.nely + 1)
    layer = mesh.nelx * mesh.nely
    for e0 in range(0, mesh.n_elem, step):
        e1 = min(mesh.n_elem, e0 + step)
        ids = np.arange(e0, e1)
        want = full[ids % layer] + (ids // layer)[:, None] * per_layer
        if not np.array_equal(edof[e0:e1], want):
            return False
    return True


@dataclass
class BoundaryConditions:
    """Fixed DOFs (sorted, unique, int64) and the nodal load vector."""

    fixed_dofs: np.ndarray
    force: np.ndarray

    def __post_init__(self):
        self.fixed_dofs = np.unique(np.asarray(self.fixed_dofs, dtype=np.int64))
        self.force = np.array(self.force, dtype=np.float64, copy=True)
        self.force[self.fixed_dofs] = 0.0

    def free_mask(self, n_dof: int) -> np.ndarray:
        m = np.ones(n_dof, dtype=bool)
        m[self.fixed_dofs] = False
        return m


@dataclass
class ProblemPreset:
    name: str
    mesh: StructuredMesh
    bcs: BoundaryConditions
    volume_fraction: float
    filter_radius: float = 1.5
    scale: float = 1.0


_BASE_DIMS = {
    "cantilever": (120, 60, 30),
    "mbb": (150, 50, 25),
    "bridge": (150, 50, 25),
    "torsion": (165, 55, 55),
}
_VOLFRAC = {"cantilever": 0.30, "mbb": 0.50, "bridge": 0.30, "torsion": 0.25}
PRESET_NAMES = tuple(_BASE_DIMS)
DESK_SCALE = 0.2


def _dims_at(name: str, scale: float) -> tuple[int, int, int]:
    out = []
    for d in _BASE_DIMS[name]:
        x = d * scale
        n = int(round(x))
        if n < 1 or abs(x - n) > 1e-9:
            raise ValueError(f"scale {scale} gives non-integer element counts for preset {name!r}")
        out.append(n)
    return tuple(out)


def _nearest_node(mesh: StructuredMesh, fx: float, fy: float, fz: float) -> int:
    return int(mesh.node_id(int(round(fx * mesh.nelx)), int(round(fy * mesh.nely)),
                            int(round(fz * mesh.nelz))))


def _face_x0_dofs(mesh: StructuredMesh) -> np.ndarray:
    nx1, ny1, nz1 = mesh.node_dims
    jj, kk = np.meshgrid(np.arange(ny1), np.arange(nz1), indexing="xy")
    nodes = np.sort(mesh.node_id(0, jj.ravel(), kk.ravel()))
    return (3 * nodes[:, None] + np.arange(3)).ravel()


def make_preset(name: str, scale: float = 1.0) -> ProblemPreset:
    """Named benchmark problems (reference mesh.py:172-232)."""
    if name not in _BASE_DIMS:
        raise ValueError(f"unknown preset {name!r}, expected one of {PRESET_NAMES}")
    mesh = StructuredMesh(*_dims_at(name, scale))
    g = mesh.node_grid()
    f = np.zeros(mesh.n_dof)
    nx, ny, nz = mesh.nelx, mesh.nely, mesh.nelz
    if name == "cantilever":
        fixed = [_face_x0_dofs(mesh)]
        f[3 * _nearest_node(mesh, 1.0, 0.5, 0.5) + 1] = -1.0
    elif name == "mbb":
        left = np.flatnonzero(g[:, 0] == 0)
        fixed = [3 * left, np.array([3 * _nearest_node(mesh, 1.0, 0.0, 0.5) + 1])]
        f[3 * _nearest_node(mesh, 0.0, 1.0, 0.5) + 1] = -1.0
    elif name == "bridge":
        ll = np.flatnonzero((g[:, 0] == 0) & (g[:, 1] == 0))
        lr = np.flatnonzero((g[:, 0] == nx) & (g[:, 1] == 0))
        fixed = [(3 * ll[:, None] + np.arange(3)).ravel(), 3 * lr + 1, 3 * lr + 2]
        top = np.flatnonzero((g[:, 1] == ny) & (g[:, 2] == int(round(0.5 * nz))))
        f[3 * top + 1] = -1.0 / top.size
    else:  # torsion
        fixed = [_face_x0_dofs(mesh)]
        top = np.flatnonzero((g[:, 0] == nx) & (g[:, 1] == ny))
        bot = np.flatnonzero((g[:, 0] == nx) & (g[:, 1] == 0))
        f[3 * top + 2] = 1.0 / top.size
        f[3 * bot + 2] = -1.0 / bot.size
    bcs = BoundaryConditions(np.concatenate(fixed), f)
    return ProblemPreset(name, mesh, bcs, _VOLFRAC[name], 1.5, scale)


def cantilever_bcs(mesh: StructuredMesh) -> BoundaryConditions:
    """Clamped x=0 face, unit -y tip load (reference mesh.py:235-246)."""
    f = np.zeros(mesh.n_dof)
    f[3 * _nearest_node(mesh, 1.0, 0.5, 0.5) + 1] = -1.0
    return BoundaryConditions(_face_x0_dofs(mesh), f)
