"""Synthetic benchmark scenes (BASELINE.json ``configs``).

* ``c1``  cantilever ~10K tets, no contact (the reference's CPU scene):
          box_grid((24,10,7),(1.2,0.5,0.35)), clamped at x=0, E=1e6.
* ``c3``  stiff beam twist, ~1M tets, no contact: box_grid((160,40,26)),
          clamped at x=0, E=2e7, initial angular velocity about the beam axis
          ramped along x (the reference's acceptance "kick" ramp,
          test_acceptance.py:139-145, turned into a twist).
* ``c2``  one stiff puffer ball (voxel SDF sphere with spikes -> Kuhn
          tets, E=2e7) resting on the ground plane, IPC barrier contact
          (``cube_drop.toml`` barrier settings).
* ``c4``  ten puffer balls in a five-plane glass tank (2 rows of 5 on the
          floor, walls and floor 0.5 dhat away, neighbouring balls 4 dhat
          apart), stiff/soft E = 2e8 / 1e7 (20x), IPC barrier contact.
          ``c4s<cells>`` is the same construction at fewer cells per ball;
          ``c4t<cells>`` packs the balls to touch (0.5 dhat), so cross-body
          vertex-triangle pairs are active from the first sweep (parity
          scenes; the reference algorithm's coupled pair rows make those
          sweeps backtrack heavily).

All scenes use gravity (0, -9.8, 0), rho = 1000, nu = 0.4, h = 1/120 and
seed 0; random-init precompute is ``Precompute.injected`` (structurally
valid, see precompute.py) wherever the reference precompute cannot run.
"""

import numpy as np

from .model import (BarrierParams, HalfSpace, MaterialParams, Model, SystemState, box_grid,
                    build_mesh, compute_z)

H = 1.0 / 120.0
# Contact scenes resolve the barrier layer: tol_dx * extent = 1% of dhat,
# the ratio of the reference's cube_drop scene (tol 1e-3 on a 0.1 m scene,
# dhat 1 cm; cube_drop.toml:10-22). A scene-level setting, like the TOML's.
CONTACT_TOL = 2.5e-5


def cantilever(divisions=(24, 10, 7), extents=(1.2, 0.5, 0.35), young=1e6):
    mesh = box_grid(divisions, extents)
    mat = MaterialParams.from_young_poisson(young, 0.4, 1000.0)
    fixed = np.flatnonzero(mesh.rest_positions[:, 0] < 1e-9)
    return Model([(mesh, mat, fixed, np.zeros(3), np.eye(3))])


def twist_state(model, h=H, omega=2.0):
    """Initial state with an angular velocity about the beam's long axis,
    ramped linearly from the clamped end (x = 0) to the free end."""
    x0 = model.initial_positions
    st = SystemState.initial(model, h)
    w = x0[:, 0] / max(x0[:, 0].max(), 1e-300)
    c = 0.5 * (x0.min(axis=0) + x0.max(axis=0))
    ry, rz = x0[:, 1] - c[1], x0[:, 2] - c[2]
    st.v[:, 1] = -omega * w * rz
    st.v[:, 2] = omega * w * ry
    st.v[model.fixed_mask] = 0.0
    return st


def puffer_ball_mesh(radius=0.5, cells=40, spikes=12, spike_amp=0.25, seed=0, center=(0, 0, 0)):
    """Kuhn-tet voxelisation of a spiky sphere SDF (cells across the
    diameter). Keeps voxels whose centre is inside the SDF."""
    rng = np.random.default_rng(seed)
    dirs = rng.standard_normal((spikes, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    ext = 2.0 * radius * (1.0 + spike_amp)
    n = int(np.ceil(cells * (1.0 + spike_amp)))
    dx = ext / n
    g = (np.arange(n) + 0.5) * dx - ext / 2
    X, Y, Zc = np.meshgrid(g, g, g, indexing="ij")
    p = np.stack([X.ravel(), Y.ravel(), Zc.ravel()], axis=1)
    r = np.linalg.norm(p, axis=1)
    u = p / np.maximum(r, 1e-12)[:, None]
    bump = np.max(np.clip(u @ dirs.T, 0.0, 1.0) ** 16, axis=1)
    inside = r <= radius * (1.0 + spike_amp * bump)
    cell = np.flatnonzero(inside.reshape(n, n, n).ravel())
    i, j, k = np.unravel_index(cell, (n, n, n))
    # Kuhn split on the shared vertex lattice
    c = np.arange(8)
    ci = i[:, None] + (c >> 2 & 1)
    cj = j[:, None] + (c >> 1 & 1)
    ck = k[:, None] + (c & 1)
    vid = (ci * (n + 1) + cj) * (n + 1) + ck
    from .model import _KUHN
    tets = vid[:, _KUHN].reshape(-1, 4)
    used, inv = np.unique(tets, return_inverse=True)
    tets = inv.reshape(-1, 4)
    li, lj, lk = np.unravel_index(used, (n + 1, n + 1, n + 1))
    verts = np.stack([li, lj, lk], axis=1) * dx - ext / 2 + np.asarray(center, dtype=np.float64)
    return build_mesh(verts, tets)


def puffer_balls(n_balls=1, cells=45, youngs=(2e7,), ncols=4, gap=0.04, walls=False, radius=0.1,
                 kappa=2e3, dhat_frac=0.01, stack_gap=0.5, stack_offset=0.0):
    """C2 (1 ball on the ground plane) / C4 (10 balls in a glass tank).

    Balls stand in columns (ncols per layer, 2 x 2 footprint); the lowest
    vertex of a bottom ball and of every stacked ball sits 0.5 dhat above
    the ground / directly above the top vertex of the ball below, so the
    barrier is active from the first sweep (plane and cross-body
    vertex-triangle pairs). Tank walls (C4) are 0.5 dhat outside the
    outermost vertices. dhat = 1% of the ball extent, kappa = 2e3
    (cube_drop.toml:18-24 shape, kappa scaled to the ball mass). Materials
    cycle through ``youngs``.
    """
    meshes = [puffer_ball_mesh(radius=radius, cells=cells, seed=b) for b in range(n_balls)]
    ext = 2.0 * radius * 1.25
    dhat = dhat_frac * ext
    shift_max = 0.35 * radius  # horizontal alignment of a stacked ball, clamped
    spacing = ext + gap + 2.0 * shift_max
    bodies, world = [], []
    tops = {}
    for b, m in enumerate(meshes):
        col, layer = b % ncols, b // ncols
        base = np.array([(col % 2) * spacing, 0.0, (col // 2) * spacing])
        x = m.rest_positions
        lo = int(np.argmin(x[:, 1]))
        if layer == 0:
            t = base - np.array([0.0, x[lo, 1], 0.0]) + np.array([0.0, 0.5 * dhat, 0.0])
        else:
            # lowest vertex 0.5 dhat above the top vertex of the ball below
            # (the whole ball stays above that height: no overlap), shifted
            # sideways to sit over it when that needs <= shift_max
            top, cen = tops[col]
            t = top - x[lo] + np.array([0.0, stack_gap * dhat, 0.0])
            if stack_offset > 0.0:
                ang = 2.0 * np.pi * (b / max(n_balls, 1))
                t[[0, 2]] = cen[[0, 2]] + stack_offset * radius * np.array([np.cos(ang), np.sin(ang)])
            else:
                off = t[[0, 2]] - cen[[0, 2]]
                n_off = float(np.linalg.norm(off))
                if n_off > shift_max:
                    t[[0, 2]] = cen[[0, 2]] + off * (shift_max / n_off)
        xw = x + t
        tops[col] = (xw[int(np.argmax(xw[:, 1]))], base)
        world.append(xw)
        mat = MaterialParams.from_young_poisson(youngs[b % len(youngs)], 0.4, 1000.0)
        bodies.append((m, mat, np.zeros(0, dtype=np.int64), t, np.eye(3)))
    planes = [HalfSpace(np.zeros(3), np.array([0.0, 1.0, 0.0]))]
    if walls:
        allx = np.vstack(world)
        lo, hi = allx.min(axis=0) - 0.5 * dhat, allx.max(axis=0) + 0.5 * dhat
        planes += [HalfSpace(np.array([lo[0], 0, 0]), np.array([1.0, 0, 0])),
                   HalfSpace(np.array([hi[0], 0, 0]), np.array([-1.0, 0, 0])),
                   HalfSpace(np.array([0, 0, lo[2]]), np.array([0, 0, 1.0])),
                   HalfSpace(np.array([0, 0, hi[2]]), np.array([0, 0, -1.0]))]
    # kappa scaled from cube_drop (0.125 kg cube, kappa 2e3) to ~500 kg balls so
    # the barrier holds a ball on a few spike tips at ~dhat/2
    return Model(bodies, planes=planes, barrier=BarrierParams(dhat=dhat, kappa=kappa))


def predictor_state(model, state):
    """z from the state's velocity; x at the (unconstrained) predictor."""
    compute_z(model, state)
    state.x = state.z.copy()
    return state


def build(name):
    """(model, state, h, description) for a named config."""
    if name == "c1":
        m = cantilever()
        st = SystemState.initial(m, H)
        return m, predictor_state(m, st), H, "C1 cantilever box_grid(24,10,7) 10,080 tets, E=1e6, no contact"
    if name == "c3":
        m = cantilever(divisions=(160, 40, 26), extents=(8.0, 2.0, 1.3), young=2e7)
        return m, predictor_state(m, twist_state(m)), H, \
            "C3 stiff beam twist box_grid(160,40,26) 998,400 tets, E=2e7, no contact"
    if name == "c2" or name.startswith("c2s"):  # c2s<cells>: fewer cells per ball
        m = puffer_balls(1, cells=45 if name == "c2" else int(name[3:]), youngs=(2e7,))
        m.tol_dx = CONTACT_TOL
        return m, predictor_state(m, SystemState.initial(m, H)), H, \
            f"C2 puffer ball {m.num_elements:,} tets on a ground plane, E=2e7, IPC barrier"
    if name == "c4" or name.startswith("c4s") or name.startswith("c4t"):
        cells = 45 if name == "c4" else int(name[3:] or 12)
        m = puffer_tank(10, cells=cells, youngs=(2e8, 1e7), ball_gap=0.5 if name.startswith("c4t") else 4.0)
        m.tol_dx = CONTACT_TOL
        desc = (f"C4 ten puffer balls {m.num_elements:,} tets in a 5-plane tank, E 2e8/1e7, IPC"
                if name == "c4" else f"C4 tank at {cells} cells/ball{' (touching)' if name.startswith('c4t') else ''}")
        return m, predictor_state(m, SystemState.initial(m, H)), H, desc
    if name.startswith("c3s"):  # scaled-down C3 for tests / CPU samples: c3s<k>
        k = int(name[3:] or 4)
        m = cantilever(divisions=(160 // k, 40 // k, max(26 // k, 2)),
                       extents=(8.0, 2.0, 1.3), young=2e7)
        return m, predictor_state(m, twist_state(m)), H, f"C3/{k} twist beam"
    raise ValueError(f"unknown scene {name!r}")


# ---------------------------------------------------------------- placement
def _point_triangle_distance(p, a, b, c):
    """Row-wise Euclidean distance from points p (n, 3) to triangles (a, b, c)
    (n, 3 each): closest-point regions (Ericson), scene setup only."""
    ab, ac, ap = b - a, c - a, p - a
    d1, d2 = np.einsum("ij,ij->i", ab, ap), np.einsum("ij,ij->i", ac, ap)
    bp = p - b
    d3, d4 = np.einsum("ij,ij->i", ab, bp), np.einsum("ij,ij->i", ac, bp)
    cp = p - c
    d5, d6 = np.einsum("ij,ij->i", ab, cp), np.einsum("ij,ij->i", ac, cp)
    va, vb, vc = d3 * d6 - d5 * d4, d5 * d2 - d1 * d6, d1 * d4 - d3 * d2
    with np.errstate(divide="ignore", invalid="ignore"):
        den = 1.0 / (va + vb + vc)
        v, w = vb * den, vc * den
        q = a + ab * v[:, None] + ac * w[:, None]
        cases = [((d1 <= 0) & (d2 <= 0), a),
                 ((d3 >= 0) & (d4 <= d3), b),
                 ((d6 >= 0) & (d5 <= d6), c),
                 ((vc <= 0) & (d1 >= 0) & (d3 <= 0), a + ab * (d1 / (d1 - d3))[:, None]),
                 ((vb <= 0) & (d2 >= 0) & (d6 <= 0), a + ac * (d2 / (d2 - d6))[:, None]),
                 ((va <= 0) & (d4 - d3 >= 0) & (d5 - d6 >= 0),
                  b + (c - b) * ((d4 - d3) / ((d4 - d3) + (d5 - d6)))[:, None])]
    done = np.zeros(len(p), dtype=bool)
    for mask, pt in cases:
        sel = mask & ~done
        q[sel] = pt[sel]
        done |= sel
    return np.linalg.norm(p - q, axis=1)


class _Surface:
    """Surface of one placed or moving body (scene setup): unique surface
    vertices, triangle corners, and KD-trees built once."""

    def __init__(self, x, tris):
        from scipy.spatial import cKDTree
        self.p = x[np.unique(tris)]
        self.tv = x[tris]
        cen = self.tv.mean(axis=1)
        self.rad = float(np.linalg.norm(self.tv - cen[:, None], axis=2).max())
        self.lo, self.hi = self.p.min(axis=0), self.p.max(axis=0)
        self.ctree, self.vtree = cKDTree(cen), cKDTree(self.p)


def _one_way_gap(src, dst, shift, reach):
    """min distance from src's vertices (moved by -shift) to dst's triangles."""
    p = src.p - shift
    box = np.maximum(np.maximum(dst.lo - p, p - dst.hi), 0.0)
    p = p[np.linalg.norm(box, axis=1) <= reach]
    if not len(p):
        return np.inf
    dvv, _ = dst.vtree.query(p)
    ub = float(dvv.min())
    near = dst.ctree.query_ball_point(p, ub + dst.rad)
    pi = np.repeat(np.arange(len(p)), [len(n) for n in near])
    if not len(pi):
        return ub
    ti = np.fromiter((t for n in near for t in n), dtype=np.int64, count=len(pi))
    tt = dst.tv[ti]
    return min(ub, float(_point_triangle_distance(p[pi], tt[:, 0], tt[:, 1], tt[:, 2]).min()))


def surface_gap(xa, tris_a, xb, tris_b, reach=np.inf):
    """Minimum vertex-triangle distance between two disjoint surfaces (both
    directions), the quantity the barrier sees (contact.py:216-240)."""
    a, b = _Surface(xa, tris_a), _Surface(xb, tris_b)
    zero = np.zeros(3)
    return min(_one_way_gap(a, b, zero, reach), _one_way_gap(b, a, zero, reach))


def place_at_gap(xa, tris_a, xb, tris_b, direction, target, lo, hi, iters=40):
    """Translation s along ``direction`` (unit) of body b, in [lo, hi], with
    surface_gap(a, b + s direction) == target (bisection; the gap shrinks as
    s decreases)."""
    d = np.asarray(direction, dtype=np.float64)
    for _ in range(iters):
        mid = 0.5 * (lo + hi)
        g = surface_gap(xa, tris_a, xb + mid * d, tris_b)
        if g > target:
            hi = mid
        else:
            lo = mid
    return hi


def puffer_tank(n_balls=10, cells=45, youngs=(2e8, 1e7), nx=5, walls=True, radius=0.1, kappa=2e3,
                dhat_frac=0.01, gap_frac=0.5, ball_gap=4.0):
    """C4: ten puffer balls on the floor of a five-plane glass tank, packed in
    an nx-wide grid so neighbouring balls touch: every ball sits gap_frac*dhat
    above the floor and gap_frac*dhat from the nearest ball already placed
    (exact vertex-triangle surface distance), the walls gap_frac*dhat outside
    the outermost vertices. Cross-body vertex-triangle pairs, plane pairs and
    wall pairs are all active from the first sweep. Materials cycle through
    ``youngs`` (stiff / soft)."""
    meshes = [puffer_ball_mesh(radius=radius, cells=cells, seed=b) for b in range(n_balls)]
    ext = 2.0 * radius * 1.25
    dhat = dhat_frac * ext
    target = ball_gap * dhat
    placed = []  # (_Surface, world positions)
    bodies = []
    for b, m in enumerate(meshes):
        i, j = b % nx, b // nx
        x = m.rest_positions
        t = np.array([0.0, gap_frac * dhat - x[:, 1].min(), 0.0])
        if placed:
            allx = np.vstack([w for _, w in placed])
            if j == 0:  # right of the row so far, slid back along -x
                axis = np.array([1.0, 0, 0])
                t[0] = allx[:, 0].max() - x[:, 0].min() + 0.05 * ext
                t[2] = placed[0][1][:, 2].mean() - x[:, 2].mean()
            else:       # behind the rows so far (above ball b - nx), slid back along -z
                axis = np.array([0, 0, 1.0])
                t[0] = placed[b - nx][1][:, 0].mean() - x[:, 0].mean()
                prev = np.vstack([w for _, w in placed[:j * nx]])
                t[2] = prev[:, 2].max() - x[:, 2].min() + 0.05 * ext
            reach = 1.01 * target  # only "gap > target?" matters
            mv = _Surface(x, m.surface_tris)  # at its rest placement; queries shift

            def gap_at(s_):
                off = t - s_ * axis
                return min(min(_one_way_gap(mv, ps, -off, reach), _one_way_gap(ps, mv, off, reach))
                           for ps, _ in placed)
            while gap_at(0.0) <= target:  # clear of the same row's balls first
                t[0] += 0.05 * ext
            lo_s, hi_s = 0.0, 0.4 * ext
            for _ in range(30):
                mid = 0.5 * (lo_s + hi_s)
                if gap_at(mid) > target:
                    lo_s = mid
                else:
                    hi_s = mid
            t = t - lo_s * axis
        placed.append((_Surface(x + t, m.surface_tris), x + t))
        mat = MaterialParams.from_young_poisson(youngs[b % len(youngs)], 0.4, 1000.0)
        bodies.append((m, mat, np.zeros(0, dtype=np.int64), t, np.eye(3)))
    planes = [HalfSpace(np.zeros(3), np.array([0.0, 1.0, 0.0]))]
    if walls:
        allx = np.vstack([w for _, w in placed])
        lo, hi = allx.min(axis=0) - gap_frac * dhat, allx.max(axis=0) + gap_frac * dhat
        planes += [HalfSpace(np.array([lo[0], 0, 0]), np.array([1.0, 0, 0])),
                   HalfSpace(np.array([hi[0], 0, 0]), np.array([-1.0, 0, 0])),
                   HalfSpace(np.array([0, 0, lo[2]]), np.array([0, 0, 1.0])),
                   HalfSpace(np.array([0, 0, hi[2]]), np.array([0, 0, -1.0]))]
    return Model(bodies, planes=planes, barrier=BarrierParams(dhat=dhat, kappa=kappa))
