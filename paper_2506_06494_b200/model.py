"""Static scene containers with the reference's attribute names.

These are the inputs that cross the drop-in boundary: the GPU
``LocalSolver`` reads only array attributes of a model object, so it accepts
this ``Model`` and the reference's ``tetsolve.assembly.Model``
(``assembly.py:40-116``) interchangeably. This module is plumbing (mesh
construction for the synthetic benchmark scenes), vectorised so that
multi-million-tet scenes build in seconds; it is not on the timed path.
"""

from dataclasses import dataclass

import numpy as np

# Faces of tet (v0,v1,v2,v3), outward for positive orientation (mesh.py:22).
_TET_FACES = np.array(((1, 2, 3), (0, 3, 2), (0, 1, 3), (0, 2, 1)))

# Kuhn split of a cell into 6 tets around the main diagonal (primitives.py:8-15).
_KUHN = np.array(((0b000, 0b100, 0b110, 0b111),
                  (0b000, 0b110, 0b010, 0b111),
                  (0b000, 0b010, 0b011, 0b111),
                  (0b000, 0b011, 0b001, 0b111),
                  (0b000, 0b001, 0b101, 0b111),
                  (0b000, 0b101, 0b100, 0b111)))


class MeshError(Exception):
    """Invalid mesh contents (mesh.py:25)."""


@dataclass(frozen=True)
class MaterialParams:
    """Lame pair + density (energy.py:18-33)."""
    mu: float
    lam: float
    density: float

    @staticmethod
    def from_young_poisson(young, poisson, density):
        mu = young / (2.0 * (1.0 + poisson))
        lam = young * poisson / ((1.0 + poisson) * (1.0 - 2.0 * poisson))
        return MaterialParams(mu=mu, lam=lam, density=density)


@dataclass(frozen=True)
class BarrierParams:
    """Log-barrier activation distance and stiffness (energy.py:36-43)."""
    dhat: float
    kappa: float


class HalfSpace:
    """Analytic contact plane with unit normal (contact.py:18-26)."""

    def __init__(self, point, normal):
        self.point = np.asarray(point, dtype=np.float64)
        n = np.asarray(normal, dtype=np.float64)
        self.normal = n / np.linalg.norm(n)


@dataclass(frozen=True)
class SceneNormalization:
    scale: float
    offset: np.ndarray


@dataclass
class TetMesh:
    """Mesh arrays (mesh.py:40-62); incidence kept as CSR, not a list."""
    rest_positions: np.ndarray
    tets: np.ndarray
    surface_tris: np.ndarray
    rest_volumes: np.ndarray
    dm_inv: np.ndarray
    vertex_masses: np.ndarray
    density: float

    @property
    def num_vertices(self):
        return self.rest_positions.shape[0]

    @property
    def num_elements(self):
        return self.tets.shape[0]


def _shape_matrices(x, tets):
    p = x[tets]
    return np.stack((p[:, 1] - p[:, 0], p[:, 2] - p[:, 0], p[:, 3] - p[:, 0]), axis=2)


def extract_surface(tets):
    """Faces used by exactly one tet, outward oriented (mesh.py:142-150)."""
    if tets.shape[0] == 0:
        return np.zeros((0, 3), dtype=np.int64)
    faces = tets[:, _TET_FACES].reshape(-1, 3)
    key = np.sort(faces, axis=1)
    _, inv, cnt = np.unique(key, axis=0, return_inverse=True, return_counts=True)
    return faces[cnt[inv.ravel()] == 1]


def build_mesh(rest_positions, tets, density=1000.0):
    """Volumes, Dm^-1, quarter-volume lumped masses, surface (mesh.py:72-133)."""
    x = np.ascontiguousarray(rest_positions, dtype=np.float64)
    tets = np.ascontiguousarray(tets, dtype=np.int64).reshape(-1, 4).copy()
    nv, ne = x.shape[0], tets.shape[0]
    if ne and (tets.min() < 0 or tets.max() >= nv):
        raise MeshError("element references a vertex out of range")
    dm = _shape_matrices(x, tets)
    vol = np.linalg.det(dm) / 6.0
    inv = np.flatnonzero(vol < 0)
    if inv.size:
        tets[inv, 2], tets[inv, 3] = tets[inv, 3].copy(), tets[inv, 2].copy()
        dm = _shape_matrices(x, tets)
        vol = np.linalg.det(dm) / 6.0
    if ne:
        if np.any(np.abs(vol) < 1e-12 * float(np.mean(np.abs(vol)))):
            raise MeshError("degenerate elements")
        dm_inv = np.linalg.inv(dm)
    else:
        dm_inv = np.zeros((0, 3, 3))
    masses = np.zeros(nv)
    if ne:
        np.add.at(masses, tets.ravel(), np.repeat(density * vol / 4.0, 4))
    return TetMesh(rest_positions=x, tets=tets, surface_tris=extract_surface(tets),
                   rest_volumes=vol, dm_inv=dm_inv, vertex_masses=masses,
                   density=float(density))


def box_grid(divisions, extents, origin=(0.0, 0.0, 0.0), density=1000.0):
    """Kuhn-split box (primitives.py:18-44), vectorised; identical vertex and
    element numbering to the reference generator."""
    nx, ny, nz = divisions
    xs = np.linspace(origin[0], origin[0] + extents[0], nx + 1)
    ys = np.linspace(origin[1], origin[1] + extents[1], ny + 1)
    zs = np.linspace(origin[2], origin[2] + extents[2], nz + 1)
    gx, gy, gz = np.meshgrid(xs, ys, zs, indexing="ij")
    verts = np.column_stack((gx.ravel(), gy.ravel(), gz.ravel()))
    i, j, k = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    i, j, k = i.ravel(), j.ravel(), k.ravel()
    c = np.arange(8)
    ci = i[:, None] + (c >> 2 & 1)
    cj = j[:, None] + (c >> 1 & 1)
    ck = k[:, None] + (c & 1)
    corner = (ci * (ny + 1) + cj) * (nz + 1) + ck           # (cells, 8)
    tets = corner[:, _KUHN].reshape(-1, 4)
    return build_mesh(verts, tets, density=density)


def incidence_csr(tets, nv):
    """Per-vertex incident (element, slot), ascending element id
    (mesh.py:114-120 order; local_solver.py:249-256 slots)."""
    tets = np.asarray(tets)
    flat = tets.ravel()
    order = np.argsort(flat, kind="stable")
    ptr = np.zeros(nv + 1, dtype=np.int64)
    np.cumsum(np.bincount(flat, minlength=nv), out=ptr[1:])
    return ptr, (order // 4).astype(np.int64), (order % 4).astype(np.int64)


def greedy_color(tets, nv):
    """First-fit greedy vertex colouring in ascending vertex id: two vertices
    sharing a tet never share a colour (mesh.py:164-178, same order and rule,
    so the colour groups of the Gauss-Seidel schedule are identical)."""
    tets = np.asarray(tets, dtype=np.int64)
    # vertex adjacency (CSR, neighbours through shared tets)
    a = np.repeat(tets, 4, axis=1).ravel()
    b = np.tile(tets, (1, 4)).ravel()
    keep = a != b
    a, b = a[keep], b[keep]
    order = np.lexsort((b, a))
    a, b = a[order], b[order]
    uniq = np.ones(a.size, dtype=bool)
    uniq[1:] = (a[1:] != a[:-1]) | (b[1:] != b[:-1])
    a, b = a[uniq], b[uniq]
    ptr = np.zeros(nv + 1, dtype=np.int64)
    np.cumsum(np.bincount(a, minlength=nv), out=ptr[1:])
    colors = np.full(nv, -1, dtype=np.int64)
    for j in range(nv):
        nb = colors[b[ptr[j]:ptr[j + 1]]]
        used = np.zeros(nb.size + 2, dtype=bool)
        nb = nb[(nb >= 0) & (nb < used.size)]
        used[nb] = True
        colors[j] = int(np.argmin(used))
    return colors


class Model:
    """Concatenated multi-body scene (assembly.py:40-116)."""

    @property
    def colors(self):
        """Greedy vertex colouring (assembly.py:110), computed on first use."""
        if getattr(self, "_colors", None) is None:
            self._colors = greedy_color(self.tets, self.num_vertices)
        return self._colors

    def __init__(self, bodies, gravity=(0.0, -9.8, 0.0), planes=(), barrier=None):
        self.bodies = []
        voff = eoff = 0
        parts = []
        for mesh, mat, fixed, translate, rotate in bodies:
            parts.append((mesh, mat, np.asarray(fixed, dtype=np.int64),
                          np.asarray(translate, dtype=np.float64),
                          np.asarray(rotate, dtype=np.float64), voff, eoff))
            self.bodies.append(parts[-1])
            voff += mesh.num_vertices
            eoff += mesh.num_elements
        self.num_vertices, self.num_elements = voff, eoff
        self.gravity = np.asarray(gravity, dtype=np.float64)
        self.planes = [p if isinstance(p, HalfSpace) else HalfSpace(*p) for p in planes]
        self.barrier = barrier
        cat = lambda xs, empty: np.concatenate(xs) if xs else empty  # noqa: E731
        P = parts
        self.rest_positions = cat([m.rest_positions for m, *_ in P], np.zeros((0, 3)))
        self.initial_positions = cat([m.rest_positions @ r.T + t for m, _, _, t, r, _, _ in P],
                                     np.zeros((0, 3)))
        self.tets = cat([m.tets + vo for m, *_, vo, _ in P], np.zeros((0, 4), np.int64))
        self.volumes = cat([m.rest_volumes for m, *_ in P], np.zeros(0))
        self.dm_inv = cat([m.dm_inv for m, *_ in P], np.zeros((0, 3, 3)))
        self.mu = cat([np.full(m.num_elements, mt.mu) for m, mt, *_ in P], np.zeros(0))
        self.lam = cat([np.full(m.num_elements, mt.lam) for m, mt, *_ in P], np.zeros(0))
        self.masses = cat([m.vertex_masses * (mt.density / m.density) for m, mt, *_ in P],
                          np.zeros(0))
        self.elem_qmass = cat([mt.density * m.rest_volumes / 4.0 for m, mt, *_ in P],
                              np.zeros(0))
        self.vertex_body = cat([np.full(m.num_vertices, k) for k, (m, *_) in enumerate(P)],
                               np.zeros(0, np.int64))
        self.tet_body = cat([np.full(m.num_elements, k) for k, (m, *_) in enumerate(P)],
                            np.zeros(0, np.int64))
        self.surface_tris = cat([m.surface_tris + vo for m, *_, vo, _ in P],
                                np.zeros((0, 3), np.int64))
        self.surface_tri_body = cat([np.full(len(m.surface_tris), k)
                                     for k, (m, *_) in enumerate(P)], np.zeros(0, np.int64))
        self.surface_vertices = np.unique(self.surface_tris) if len(self.surface_tris) \
            else np.zeros(0, dtype=np.int64)
        self.fixed_mask = np.zeros(self.num_vertices, dtype=bool)
        for _, _, fixed, _, _, vo, _ in P:
            self.fixed_mask[fixed + vo] = True
        self.free_mask = ~self.fixed_mask
        self._finish()

    def _finish(self):
        x0 = self.initial_positions
        if len(x0):
            lo = x0.min(axis=0)
            extent = float((x0.max(axis=0) - lo).max())
        else:
            lo, extent = np.zeros(3), 1.0
        if extent <= 0:
            extent = 1.0
        self.normalization = SceneNormalization(scale=1.0 / extent, offset=-lo / extent)

    @classmethod
    def from_arrays(cls, arrays, prefix="model_"):
        """Rebuild from the golden-fixture layout (tests/golden/make_goldens.py)."""
        a = {k[len(prefix):]: v for k, v in arrays.items() if k.startswith(prefix)}
        self = cls.__new__(cls)
        for key in ("rest_positions", "initial_positions", "tets", "volumes", "dm_inv",
                    "mu", "lam", "masses", "elem_qmass", "fixed_mask", "vertex_body",
                    "tet_body", "surface_tris", "surface_tri_body", "surface_vertices",
                    "gravity"):
            setattr(self, key, np.array(a[key]))
        self.num_vertices = self.rest_positions.shape[0]
        self.num_elements = self.tets.shape[0]
        self.free_mask = ~self.fixed_mask
        self.planes = [HalfSpace(p, n) for p, n in zip(a["plane_points"], a["plane_normals"])]
        self.barrier = BarrierParams(*map(float, a["barrier"])) if a["barrier"].size else None
        self.bodies = list(a["body_vertex_offsets"])
        self._colors = np.array(a["colors"]) if "colors" in a else None
        self._finish()
        return self

    def dx_norm(self, dx):
        """assembly.py:118-120."""
        return float(self.normalization.scale * np.linalg.norm(dx))


@dataclass
class SystemState:
    """Per-frame state (assembly.py:131-144)."""
    x: np.ndarray
    x_prev: np.ndarray
    v: np.ndarray
    z: np.ndarray
    h: float
    rotations: np.ndarray = None

    @staticmethod
    def initial(model, h):
        x0 = np.array(model.initial_positions, dtype=np.float64)
        return SystemState(x=x0.copy(), x_prev=x0.copy(), v=np.zeros_like(x0),
                           z=x0.copy(), h=float(h))


def compute_z(model, state):
    """Inertia target, Dirichlet vertices pinned (assembly.py:165-180)."""
    h = state.h
    z = state.x_prev + h * state.v + h * h * np.broadcast_to(model.gravity, state.x_prev.shape)
    fm = np.asarray(model.fixed_mask)
    z[fm] = state.x_prev[fm]
    state.z = z
    return z


def step_velocity_update(model, state, x_new):
    """assembly.py:346-351."""
    state.v = (x_new - state.x_prev) / state.h
    state.x_prev = x_new.copy()
    state.x = x_new.copy()
    return state
