"""CPU oracle for the JGS2 runtime iteration -- TEST INFRASTRUCTURE ONLY.

This module restates, in numpy/SciPy, the reference package's (``tetsolve``
0.1.0, pure Python) runtime path for ``LocalSolver.sweep`` /
``LocalSolver.outer_solve`` in ``subspace="corotated_cubature"``,
``mode="jacobi"`` (``pkg/src/tetsolve/local_solver.py:606-721``). Each function
cites the reference file:line it follows (paths relative to
``/root/reference/pkg/src/tetsolve``).

Rules:
  * Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
    ``cpu_baseline`` / ``--impl reference`` leg may import this module, and only
    as the checker or the timed CPU baseline.  The product package
    (``paper_2506_06494_b200``) never imports it; there is no CPU fallback.
  * Parity pinning: ``tests/test_oracle_golden.py`` checks this oracle against
    golden fixtures produced by running the reference itself
    (``tests/golden/make_goldens.py``) on the bundled scenes and the C1 config.
  * Third-party arithmetic on the path is SciPy SuperLU (``splu``, scipy 1.18.1
    here), used exactly as the reference uses it (``subspace.py:126-130``,
    ``local_solver.py:115-126``); numpy LAPACK (gesv/syevd/gesdd/getrf).

The model argument is duck-typed: any object with the reference ``Model``
array attributes (``assembly.py:40-116``) works, including the product's
``paper_2506_06494_b200.model.Model`` and the reference's own ``Model``.
"""

from dataclasses import dataclass, field
import time

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla


class Infeasible(Exception):
    """A barrier distance reached <= 0 (reference ``energy.FeasibilityError``,
    energy.py:14, raised at energy.py:211-212)."""


# ===================================================================== physics
def _stack_cols(a, b, c):
    return np.stack((a, b, c), axis=-1)


def shape_weights(dm_inv):
    """W (..., 4, 3) with dF[:, j]/dx_m = W[m, j] I (energy.py:152-157)."""
    w = np.empty(dm_inv.shape[:-2] + (4, 3))
    w[..., 1:, :] = dm_inv
    w[..., 0, :] = -dm_inv.sum(axis=-2)
    return w


def deformation_gradients(xe, dm_inv):
    """F = Ds Dm^-1 for element corner positions xe (..., 4, 3) (energy.py:53-59)."""
    xe = np.asarray(xe, dtype=np.float64)
    ds = _stack_cols(xe[..., 1, :] - xe[..., 0, :],
                     xe[..., 2, :] - xe[..., 0, :],
                     xe[..., 3, :] - xe[..., 0, :])
    return ds @ dm_inv


def snh_constants(mu, lam):
    """Stable Neo-Hookean reparameterisation (energy.py:62-68)."""
    mu = np.asarray(mu, dtype=np.float64)
    lam = np.asarray(lam, dtype=np.float64)
    mu_s = 4.0 * mu / 3.0
    lam_s = lam + 5.0 * mu / 6.0
    return mu_s, lam_s, 1.0 + 0.75 * mu_s / lam_s


def cofactor(F):
    """Columns are cross products of the other two columns (energy.py:71-76)."""
    c0 = np.cross(F[..., :, 1], F[..., :, 2])
    c1 = np.cross(F[..., :, 2], F[..., :, 0])
    c2 = np.cross(F[..., :, 0], F[..., :, 1])
    return _stack_cols(c0, c1, c2)


def snh_psi(F, mu, lam):
    """Energy density (energy.py:79-86)."""
    mu_s, lam_s, alpha = snh_constants(mu, lam)
    ic = np.einsum("...ij,...ij->...", F, F)
    J = np.linalg.det(F)
    psi0 = -0.5 * mu_s * np.log(4.0) + 0.5 * lam_s * (1.0 - alpha) ** 2
    return (0.5 * mu_s * (ic - 3.0) - 0.5 * mu_s * np.log(ic + 1.0)
            + 0.5 * lam_s * (J - alpha) ** 2 - psi0)


def snh_stress(F, mu, lam):
    """First Piola-Kirchhoff stress (energy.py:89-97)."""
    mu_s, lam_s, alpha = snh_constants(mu, lam)
    ic = np.einsum("...ij,...ij->...", F, F)
    J = np.linalg.det(F)
    return ((mu_s * (1.0 - 1.0 / (ic + 1.0)))[..., None, None] * F
            + (lam_s * (J - alpha))[..., None, None] * cofactor(F))


def _skew(v):
    z = np.zeros(v.shape[:-1])
    return np.stack([np.stack([z, -v[..., 2], v[..., 1]], -1),
                     np.stack([v[..., 2], z, -v[..., 0]], -1),
                     np.stack([-v[..., 1], v[..., 0], z], -1)], -2)


def snh_hessian9(F, mu, lam):
    """d2psi/dF2 in column-stacked vec(F) order (energy.py:110-141)."""
    F = np.asarray(F, dtype=np.float64)
    lead = F.shape[:-2]
    mu_s, lam_s, alpha = (np.broadcast_to(c, lead) for c in snh_constants(mu, lam))
    ic = np.einsum("...ij,...ij->...", F, F)
    J = np.linalg.det(F)
    fv = np.swapaxes(F, -1, -2).reshape(lead + (9,))
    gv = np.swapaxes(cofactor(F), -1, -2).reshape(lead + (9,))
    H = np.zeros(lead + (9, 9))
    d = np.arange(9)
    H[..., d, d] = (mu_s * (1.0 - 1.0 / (ic + 1.0)))[..., None]
    H += (2.0 * mu_s / (ic + 1.0) ** 2)[..., None, None] * fv[..., :, None] * fv[..., None, :]
    H += lam_s[..., None, None] * gv[..., :, None] * gv[..., None, :]
    s = (lam_s * (J - alpha))[..., None, None]
    k0, k1, k2 = (_skew(F[..., :, c]) for c in range(3))
    # d cof / dF block-skew structure (energy.py:130-140)
    for (bi, bj, blk) in ((0, 1, -k2), (0, 2, k1), (1, 0, k2),
                          (1, 2, -k0), (2, 0, -k1), (2, 1, k0)):
        H[..., 3 * bi:3 * bi + 3, 3 * bj:3 * bj + 3] += s * blk
    return H


def clamp_psd(h):
    """Eigenvalue clamp to the PSD cone (energy.py:144-149)."""
    sym = 0.5 * (h + np.swapaxes(h, -1, -2))
    w, v = np.linalg.eigh(sym)
    return (v * np.maximum(w, 0.0)[..., None, :]) @ np.swapaxes(v, -1, -2)


def element_terms(xe, dm_inv, vol, mu, lam, hessian=True, project=False):
    """(energy, 12-gradient, 12x12 Hessian) per element (energy.py:169-189)."""
    F = deformation_gradients(xe, dm_inv)
    e = vol * snh_psi(F, mu, lam)
    P = snh_stress(F, mu, lam)
    W = shape_weights(dm_inv)
    g = vol[:, None] * np.einsum("emj,erj->emr", W, P).reshape(-1, 12)
    if not hessian:
        return e, g, None
    h9 = snh_hessian9(F, mu, lam).reshape(-1, 3, 3, 3, 3)
    h12 = np.einsum("emj,ejrks,enk->emrns", W, h9, W).reshape(-1, 12, 12)
    h12 *= vol[:, None, None]
    if project:
        h12 = clamp_psd(h12)
    return e, g, h12


def element_energies(xe, dm_inv, vol, mu, lam):
    """energy.py:192-194."""
    return vol * snh_psi(deformation_gradients(xe, dm_inv), mu, lam)


def barrier(d, dhat, kappa):
    """(B, B', B'') of the clamped log barrier (energy.py:205-221)."""
    if d <= 0.0:
        raise Infeasible(f"barrier distance {d} <= 0")
    if d >= dhat:
        return 0.0, 0.0, 0.0
    gap = d - dhat
    ln = np.log(d / dhat)
    return (float(-kappa * gap * gap * ln),
            float(-kappa * (2.0 * gap * ln + gap * gap / d)),
            float(-kappa * (2.0 * ln + 4.0 * gap / d - gap * gap / (d * d))))


# ===================================================================== contact
PLANE, TRIANGLE = 0, 1


@dataclass
class Pairs:
    """Active pair table (contact.ContactPair rows, contact.py:29-42)."""
    kind: np.ndarray      # (P,) 0 plane / 1 triangle
    vertex: np.ndarray    # (P,)
    tri: np.ndarray       # (P, 3), -1 for planes
    plane: np.ndarray     # (P,), -1 for triangles
    d: np.ndarray         # (P,)
    bary: np.ndarray      # (P, 3)

    def __len__(self):
        return int(self.kind.size)

    def stencil(self, k):
        if self.kind[k] == PLANE:
            return np.array([self.vertex[k]])
        return np.concatenate(([self.vertex[k]], self.tri[k]))

    def as_rows(self):
        """(P, 10) rows in the golden-fixture layout."""
        out = np.zeros((len(self), 10))
        out[:, 0] = self.kind
        out[:, 1] = self.vertex
        tri = self.kind == TRIANGLE
        out[tri, 2:5] = self.tri[tri]
        out[:, 5] = self.plane
        out[:, 6] = self.d
        out[tri, 7:10] = self.bary[tri]
        return out


def closest_points(p, tri):
    """All-pairs closest points, region-classified (contact.py:162-213).

    Returns (dist (n, m), bary (n, m, 3)) with exact zeros in clamped regions;
    regions are assigned in the reference's fixed precedence order.
    """
    a, b, c = tri[:, 0], tri[:, 1], tri[:, 2]
    ab, ac = b - a, c - a
    ap = p[:, None, :] - a[None]
    bp = p[:, None, :] - b[None]
    cp = p[:, None, :] - c[None]
    dot = lambda e, r: np.einsum("mk,nmk->nm", e, r)  # noqa: E731
    d1, d2 = dot(ab, ap), dot(ac, ap)
    d3, d4 = dot(ab, bp), dot(ac, bp)
    d5, d6 = dot(ab, cp), dot(ac, cp)
    vc = d1 * d4 - d3 * d2
    vb = d5 * d2 - d1 * d6
    va = d3 * d6 - d5 * d4
    bary = np.zeros(d1.shape + (3,))
    open_ = np.ones(d1.shape, dtype=bool)

    def take(mask, b0, b1, b2):
        sel = mask & open_
        for k, val in enumerate((b0, b1, b2)):
            bary[sel, k] = np.broadcast_to(val, d1.shape)[sel]
        open_[sel] = False

    with np.errstate(divide="ignore", invalid="ignore"):
        take((d1 <= 0) & (d2 <= 0), 1.0, 0.0, 0.0)
        take((d3 >= 0) & (d4 <= d3), 0.0, 1.0, 0.0)
        take((d6 >= 0) & (d5 <= d6), 0.0, 0.0, 1.0)
        t = d1 / (d1 - d3)
        take((vc <= 0) & (d1 >= 0) & (d3 <= 0), 1.0 - t, t, 0.0)
        t = d2 / (d2 - d6)
        take((vb <= 0) & (d2 >= 0) & (d6 <= 0), 1.0 - t, 0.0, t)
        t = (d4 - d3) / ((d4 - d3) + (d5 - d6))
        take((va <= 0) & (d4 - d3 >= 0) & (d5 - d6 >= 0), 0.0, 1.0 - t, t)
        den = va + vb + vc
        take(np.ones_like(open_), va / den, vb / den, vc / den)
    q = (np.einsum("nm,mk->nmk", bary[..., 0], a)
         + np.einsum("nm,mk->nmk", bary[..., 1], b)
         + np.einsum("nm,mk->nmk", bary[..., 2], c))
    return np.linalg.norm(p[:, None, :] - q, axis=2), bary


# Exact spatial pruning of the vertex-triangle candidates (fixture
# generation at scale, tests/golden/make_scale_goldens.py): the narrowphase
# and the row-major order are the brute-force ones; only (vertex, triangle)
# combinations that cannot be within dhat are skipped. Off by default.
PRUNE = False


def _pruned_candidates(xs, tris_x, dhat):
    """Superset of the (vertex row, triangle row) pairs with distance < dhat:
    |p - centroid| < dhat + circumradius bound, row-major order."""
    from scipy.spatial import cKDTree
    cen = tris_x.mean(axis=1)
    rad = np.linalg.norm(tris_x - cen[:, None], axis=2).max(axis=1)
    tree = cKDTree(xs)
    lists = tree.query_ball_point(cen, dhat * (1.0 + 1e-9) + rad * (1.0 + 1e-12) + 1e-300)
    ti = np.repeat(np.arange(len(cen)), [len(l) for l in lists])
    vi = np.fromiter((v for l in lists for v in l), dtype=np.int64, count=ti.size)
    order = np.lexsort((ti, vi))
    return vi[order], ti[order]


def find_pairs(model, x):
    """Brute-force active set (assembly.py:122-128 -> contact.py:216-240).

    Plane pairs first (plane order, ascending surface vertex), then
    cross-body vertex-triangle pairs in row-major (vertex, triangle) order.
    With PRUNE the same narrowphase runs per vertex on its candidate
    triangles only (identical output, checked against brute force in
    tests/test_oracle_golden.py).
    """
    empty = Pairs(*(np.zeros(0, dtype=np.int64) for _ in range(2)),
                  np.zeros((0, 3), dtype=np.int64), np.zeros(0, dtype=np.int64),
                  np.zeros(0), np.zeros((0, 3)))
    if model.barrier is None:
        return empty
    dhat = model.barrier.dhat
    sv = np.asarray(model.surface_vertices)
    rows = {k: [] for k in ("kind", "vertex", "tri", "plane", "d", "bary")}
    for pi, pl in enumerate(model.planes):
        dist = (x[sv] - pl.point) @ pl.normal
        for k in np.flatnonzero(dist < dhat):
            rows["kind"].append(PLANE)
            rows["vertex"].append(int(sv[k]))
            rows["tri"].append((-1, -1, -1))
            rows["plane"].append(pi)
            rows["d"].append(float(dist[k]))
            rows["bary"].append((0.0, 0.0, 0.0))
    st = np.asarray(model.surface_tris)
    if len(st) and len(sv) and PRUNE:
        vb, tb = np.asarray(model.vertex_body), np.asarray(model.surface_tri_body)
        vi, ti = _pruned_candidates(x[sv], x[st], dhat)
        keep = vb[sv[vi]] != tb[ti]
        vi, ti = vi[keep], ti[keep]
        starts = np.flatnonzero(np.r_[True, vi[1:] != vi[:-1]]) if vi.size else np.zeros(0, np.int64)
        ends = np.r_[starts[1:], vi.size]
        for a, b in zip(starts, ends):
            v, tt = vi[a], ti[a:b]
            dist, bary = closest_points(x[sv[v:v + 1]], x[st[tt]])
            for j in np.flatnonzero(dist[0] < dhat):
                rows["kind"].append(TRIANGLE)
                rows["vertex"].append(int(sv[v]))
                rows["tri"].append(tuple(int(w) for w in st[tt[j]]))
                rows["plane"].append(-1)
                rows["d"].append(float(dist[0, j]))
                rows["bary"].append(tuple(bary[0, j]))
    elif len(st) and len(sv):
        dist, bary = closest_points(x[sv], x[st])
        cross = (np.asarray(model.vertex_body)[sv][:, None]
                 != np.asarray(model.surface_tri_body)[None, :])
        for vi, ti in zip(*np.nonzero((dist < dhat) & cross)):
            rows["kind"].append(TRIANGLE)
            rows["vertex"].append(int(sv[vi]))
            rows["tri"].append(tuple(int(w) for w in st[ti]))
            rows["plane"].append(-1)
            rows["d"].append(float(dist[vi, ti]))
            rows["bary"].append(tuple(bary[vi, ti]))
    if not rows["kind"]:
        return empty
    return Pairs(np.array(rows["kind"]), np.array(rows["vertex"]),
                 np.array(rows["tri"], dtype=np.int64), np.array(rows["plane"]),
                 np.array(rows["d"]), np.array(rows["bary"], dtype=np.float64))


def _dist_point_point(x, y):
    """contact.py:51-59."""
    r = x - y
    d = np.linalg.norm(r)
    u = r / d
    k = (np.eye(3) - np.outer(u, u)) / d
    return d, np.concatenate((u, -u)), np.block([[k, -k], [-k, k]])


def _dist_point_edge(x, a, b):
    """Point-to-line distance |w x e| / |e| (contact.py:62-92)."""
    w, e = x - a, b - a
    m = np.cross(w, e)
    r, el = np.linalg.norm(m), np.linalg.norm(e)
    mh = m / r
    I3 = np.eye(3)
    jw = np.hstack((I3, -I3, np.zeros((3, 3))))
    je = np.hstack((np.zeros((3, 3)), -I3, I3))
    jm = -_skew(e) @ jw + _skew(w) @ je
    gm = mh / el
    grad = jm.T @ gm + je.T @ (-(r / el ** 3) * e)
    bmm = (I3 - np.outer(mh, mh)) / (r * el)
    bme = -np.outer(mh, e) / el ** 3
    bee = r * (3.0 * np.outer(e, e) / el ** 5 - I3 / el ** 3)
    hess = (jm.T @ bmm @ jm + jm.T @ bme @ je + je.T @ bme.T @ jm
            + je.T @ bee @ je)
    sk = _skew(gm)
    hess += jw.T @ (-sk) @ je + je.T @ sk @ jw
    return r / el, grad, hess


def _dist_point_face(x, a, b, c):
    """Unsigned distance to the triangle's plane (contact.py:95-127)."""
    w, u, v = x - a, b - a, c - a
    n = np.cross(u, v)
    ln = np.linalg.norm(n)
    nh = n / ln
    s = w @ nh
    I3, Z = np.eye(3), np.zeros((3, 3))
    jw = np.hstack((I3, -I3, Z, Z))
    ju = np.hstack((Z, -I3, I3, Z))
    jv = np.hstack((Z, -I3, Z, I3))
    jn = -_skew(v) @ ju + _skew(u) @ jv
    gn = (w - s * nh) / ln
    grad = jw.T @ nh + jn.T @ gn
    pn = (I3 - np.outer(nh, nh)) / ln
    bnn = (-np.outer(w, nh) - np.outer(nh, w) - s * I3
           + 3.0 * s * np.outer(nh, nh)) / ln ** 2
    hess = jw.T @ pn @ jn + jn.T @ pn @ jw + jn.T @ bnn @ jn
    sk = _skew(gn)
    hess += ju.T @ (-sk) @ jv + jv.T @ sk @ ju
    sign = 1.0 if s >= 0.0 else -1.0
    return abs(s), sign * grad, sign * hess


def _embed(g_sub, h_sub, slots):
    """contact.py:130-139."""
    g = np.zeros(12)
    h = np.zeros((12, 12))
    idx = np.concatenate([np.arange(3 * s, 3 * s + 3) for s in slots])
    g[idx] = g_sub
    h[np.ix_(idx, idx)] = h_sub
    return g, h


def pair_distance(model, x, pairs, k):
    """(d, grad, hess) of one pair's distance (contact.py:142-159, 243-251)."""
    if pairs.kind[k] == PLANE:
        pl = model.planes[pairs.plane[k]]
        return float((x[pairs.vertex[k]] - pl.point) @ pl.normal), pl.normal.copy(), \
            np.zeros((3, 3))
    p = x[pairs.vertex[k]]
    corners = x[pairs.tri[k]]
    nz = np.flatnonzero(pairs.bary[k] != 0.0)
    if len(nz) == 1:
        d, g, h = _dist_point_point(p, corners[nz[0]])
        return (d, *_embed(g, h, (0, 1 + nz[0])))
    if len(nz) == 2:
        d, g, h = _dist_point_edge(p, corners[nz[0]], corners[nz[1]])
        return (d, *_embed(g, h, (0, 1 + nz[0], 1 + nz[1])))
    return _dist_point_face(p, *corners)


def pair_terms(model, x, pairs, k, project=False):
    """Barrier energy, stencil gradient and Hessian (contact.py:254-263)."""
    d, gd, hd = pair_distance(model, x, pairs, k)
    b, db, ddb = barrier(d, model.barrier.dhat, model.barrier.kappa)
    h = ddb * np.outer(gd, gd) + db * hd
    return b, db * gd, (clamp_psd(h) if project else h)


def pair_live_distance(model, x, pairs, k):
    """Distance recomputed from scratch (contact.py:266-284)."""
    if pairs.kind[k] == PLANE:
        pl = model.planes[pairs.plane[k]]
        return float((x[pairs.vertex[k]] - pl.point) @ pl.normal)
    dist, _ = closest_points(x[pairs.vertex[k]][None], x[pairs.tri[k]][None])
    return float(dist[0, 0])


# ============================================================ global energy
def total_energy(model, z, h, x, pairs):
    """Incremental potential (assembly.py:183-192)."""
    el = float(np.sum(element_energies(x[model.tets], model.dm_inv, model.volumes,
                                       model.mu, model.lam)))
    diff = x - z
    inert = float(0.5 * np.sum(model.masses * np.einsum("ij,ij->i", diff, diff)) / h ** 2)
    bar = 0.0
    for k in range(len(pairs)):
        bar += barrier(pair_live_distance(model, x, pairs, k),
                       model.barrier.dhat, model.barrier.kappa)[0]
    return el + inert + bar


def feasibility_cap(model, x, dx):
    """Conservative step cap (assembly.py:263-291)."""
    if model.barrier is None or not len(model.surface_vertices):
        return 1.0
    cap = 1.0
    sv = np.asarray(model.surface_vertices)
    for pl in model.planes:
        d = (x[sv] - pl.point) @ pl.normal
        rate = -(dx[sv] @ pl.normal)
        mv = rate > 0
        if np.any(mv):
            cap = min(cap, 0.9 * float(np.min(d[mv] / rate[mv])))
    st = np.asarray(model.surface_tris)
    if len(model.bodies) > 1 and len(st) and PRUNE:
        cap = min(cap, _pruned_pair_cap(model, x, dx, sv, st, cap))
    elif len(model.bodies) > 1 and len(st):
        dist, _ = closest_points(x[sv], x[st])
        cross = (np.asarray(model.vertex_body)[sv][:, None]
                 != np.asarray(model.surface_tri_body)[None, :])
        dist = np.where(cross, dist, np.inf)
        rate = (np.linalg.norm(dx[sv], axis=1)[:, None]
                + np.linalg.norm(dx[st], axis=2).max(axis=1)[None, :])
        ok = rate > 1e-30
        if np.any(ok):
            cap = min(cap, 0.9 * float(np.min(dist[ok] / rate[ok])))
    return max(cap, 0.0)


def _pruned_pair_cap(model, x, dx, sv, st, ub):
    """0.9 min dist/rate over cross pairs (assembly.py:280-290), skipping only
    pairs that provably cannot go below the upper bound ``ub``: dist >=
    |p - centroid| - circumradius and rate <= |dx_v| + max_t |dx_t|. The
    surviving pairs use the brute-force arithmetic, so the min is identical."""
    from scipy.spatial import cKDTree
    p, tri = x[sv], x[st]
    sp_v = np.linalg.norm(dx[sv], axis=1)
    sp_t = np.linalg.norm(dx[st], axis=2).max(axis=1)
    cen = tri.mean(axis=1)
    rad = float(np.linalg.norm(tri - cen[:, None], axis=2).max())
    r = (ub / 0.9) * (sp_v + sp_t.max()) * (1.0 + 1e-9) + rad * (1.0 + 1e-12) + 1e-300
    lists = cKDTree(cen).query_ball_point(p, r)
    vb, tb = np.asarray(model.vertex_body)[sv], np.asarray(model.surface_tri_body)
    best = np.inf
    for vi, tl in enumerate(lists):
        if not tl:
            continue
        tt = np.asarray(tl, dtype=np.int64)
        tt = tt[tb[tt] != vb[vi]]
        if not tt.size:
            continue
        dist, _ = closest_points(p[vi:vi + 1], tri[tt])
        rate = sp_v[vi] + sp_t[tt]
        ok = rate > 1e-30
        if np.any(ok):
            best = min(best, float(np.min(dist[0][ok] / rate[ok])))
    return 0.9 * best if np.isfinite(best) else np.inf


# ============================================================ rest factor
def rest_hessian(model, h_ref):
    """Dirichlet-eliminated rest Hessian M/h^2 + PSD elastic
    (subspace.py:48-57 -> assembly.py:195-260)."""
    x0 = np.asarray(model.rest_positions, dtype=np.float64)
    nv = x0.shape[0]
    n = 3 * nv
    _, _, h_el = element_terms(x0[model.tets], model.dm_inv, model.volumes,
                               model.mu, model.lam, hessian=True, project=True)
    dof = (3 * model.tets[:, :, None] + np.arange(3)).reshape(-1, 12)
    rows = [np.repeat(dof, 12, axis=1).ravel(), np.arange(n)]
    cols = [np.tile(dof, (1, 12)).ravel(), np.arange(n)]
    vals = [h_el.ravel(), np.repeat(model.masses / h_ref ** 2, 3)]
    H = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(n, n)).tocsr()
    fixed = np.flatnonzero(np.repeat(model.fixed_mask, 3))
    if fixed.size:
        keep = np.setdiff1d(np.arange(n), fixed)
        mask = sp.csr_matrix((np.ones(keep.size), (keep, keep)), shape=(n, n))
        H = mask @ H @ mask + sp.csr_matrix((np.ones(fixed.size), (fixed, fixed)),
                                            shape=(n, n))
    return H


def rest_factor(hbar):
    """SuperLU with SciPy defaults (subspace.py:126-130)."""
    return spla.splu(hbar.tocsc())


# ============================================================ rotations
def vertex_rotations(model, x):
    """Polar factors of volume-weighted incident F sums (subspace.py:206-231)."""
    nv = model.num_vertices
    rot = np.tile(np.eye(3), (nv, 1, 1))
    if len(model.tets) == 0:
        return rot
    fw = deformation_gradients(x[model.tets], model.dm_inv) * model.volumes[:, None, None]
    acc = np.zeros((nv, 3, 3))
    np.add.at(acc, model.tets.ravel(), np.repeat(fw, 4, axis=0))
    nrm = np.linalg.norm(acc, axis=(1, 2))
    ok = nrm > 1e-12
    if not np.any(ok):
        return rot
    u, s, vt = np.linalg.svd(acc[ok])
    u[:, :, 2] *= np.sign(np.linalg.det(u @ vt))[:, None]
    r = u @ vt
    r[s[:, 0] <= 1e-12 * np.maximum(nrm[ok], 1.0)] = np.eye(3)
    rot[ok] = r
    return rot


# ============================================================ precompute packs
@dataclass
class Packs:
    """Flat per-vertex runtime tables (local_solver.py:243-303)."""
    free: np.ndarray
    valence: np.ndarray
    gbar: np.ndarray        # (nv, 3, 3)
    gbar_rows: np.ndarray   # (nv, 3, 3*gmax)
    group: np.ndarray       # (nv, gmax)
    cub_ids: np.ndarray     # (nv, s)
    cub_w: np.ndarray
    cub_valid: np.ndarray
    cub_rows: np.ndarray    # (nv, s, 4, 3, 3)
    cub_verts: np.ndarray   # (nv, s, 4)
    vrows: dict             # vertex -> {w: (3,3)}


def build_packs(model, pre):
    """Pack precompute arrays (golden layout / product ``Precompute``)."""
    nv = model.num_vertices
    free = np.flatnonzero(~np.asarray(model.fixed_mask))
    valence = np.bincount(np.asarray(model.tets).ravel(), minlength=nv)
    verts = np.asarray(pre["vertices"])
    index = {int(v): k for k, v in enumerate(verts)}
    gmax = pre["group"].shape[1]
    gbar = np.zeros((nv, 3, 3))
    grows = np.zeros((nv, 3, 3 * gmax))
    group = np.zeros((nv, gmax), dtype=np.int64)
    vrows = {}
    cptr = np.asarray(pre["cub_ptr"])
    smax = int(max((cptr[index[int(v)] + 1] - cptr[index[int(v)]] for v in free),
                   default=0))
    cub_ids = np.zeros((nv, smax), dtype=np.int64)
    cub_w = np.zeros((nv, smax))
    cub_valid = np.zeros((nv, smax), dtype=bool)
    cub_rows = np.zeros((nv, smax, 4, 3, 3))
    cub_verts = np.zeros((nv, smax, 4), dtype=np.int64)
    rptr = np.asarray(pre["vrows_ptr"])
    for v in free:
        k = index[int(v)]
        gbar[v] = pre["gbar"][k]
        grp = pre["group"][k]
        ng = int(np.count_nonzero(grp >= 0))
        grows[v, :, :3 * ng] = pre["gbar_rows"][k][:, :3 * ng]
        group[v, :ng] = grp[:ng]
        keys = pre["vrows_keys"][rptr[k]:rptr[k + 1]]
        blocks = pre["vrows"][rptr[k]:rptr[k + 1]]
        vrows[int(v)] = {int(w): blocks[j] for j, w in enumerate(keys)}
        elems = pre["cub_elems"][cptr[k]:cptr[k + 1]]
        wts = pre["cub_weights"][cptr[k]:cptr[k + 1]]
        for j, e in enumerate(elems):
            corner = model.tets[e]
            missing = [int(w) for w in corner if int(w) not in vrows[int(v)]]
            if missing:
                raise KeyError(f"basis at vertex {v} lacks rows for {missing} "
                               f"of cubature element {int(e)}")
            cub_ids[v, j] = e
            cub_w[v, j] = wts[j]
            cub_valid[v, j] = True
            cub_verts[v, j] = corner
            cub_rows[v, j] = np.stack([vrows[int(v)][int(w)] for w in corner])
    return Packs(free, valence, gbar, grows, group, cub_ids, cub_w, cub_valid,
                 cub_rows, cub_verts, vrows)


# ============================================================ solver
@dataclass
class OracleConfig:
    """SolverConfig subset on the path (local_solver.py:38-56)."""
    tol_dx: float = 1e-3
    max_outer: int = 500
    local_line_search: bool = True
    track_energy: bool = True
    max_halvings: int = 30
    alpha_floor: float = 1e-6
    mode: str = "jacobi"          # or "gauss_seidel" (local_solver.py:627-649)


@dataclass
class OracleStats:
    """IterationStats (local_solver.py:59-69)."""
    energies: list = field(default_factory=list)
    dx_norms: list = field(default_factory=list)
    grad_norms: list = field(default_factory=list)
    max_local_steps: list = field(default_factory=list)
    line_search_activations: list = field(default_factory=list)
    wall_ms: list = field(default_factory=list)
    outer_iterations: int = 0
    wall_seconds: float = 0.0
    converged: bool = False


class OracleSolver:
    """Jacobi corotated-cubature sweeps on CPU (local_solver.py:214-721)."""

    def __init__(self, model, pre, h_ref, config=None, factor=None):
        self.m = model
        self.cfg = config or OracleConfig()
        self.p = build_packs(model, pre)
        self.factor = factor if factor is not None else rest_factor(rest_hessian(model, h_ref))
        rest = np.asarray(model.rest_positions, dtype=np.float64)
        _, _, self.h_rest = element_terms(rest[model.tets], model.dm_inv, model.volumes,
                                          model.mu, model.lam, project=True)

    # ---------------------------------------------------------- fields
    def assembled_field(self, x, z, h, pairs):
        """local_solver.py:306-323 with cubature.py:37-60, 83-90."""
        m = self.m
        _, g, _ = element_terms(x[m.tets], m.dm_inv, m.volumes, m.mu, m.lam,
                                hessian=False)
        g = g + m.elem_qmass[:, None] * ((x - z) / h ** 2)[m.tets].reshape(-1, 12)
        out = np.zeros((m.num_vertices, 3))
        np.add.at(out, m.tets.ravel(), g.reshape(-1, 4, 3).reshape(-1, 3))
        iso = self.p.valence == 0
        if np.any(iso):
            out[iso] += (m.masses[iso] / h ** 2)[:, None] * (x[iso] - z[iso])
        for k in range(len(pairs)):
            _, gp, _ = pair_terms(m, x, pairs, k)
            out[pairs.stencil(k)] += gp.reshape(-1, 3)
        return out

    def collect(self, rot, g_asm):
        """q = Hbar^-1 (R^T g), fixed rows zeroed (local_solver.py:115-126)."""
        y = np.einsum("wba,wb->wa", rot, g_asm)
        y[np.asarray(self.m.fixed_mask)] = 0.0
        return self.factor.solve(y.ravel()).reshape(-1, 3)

    def corrections(self, x, verts, rot):
        """Cubature-sampled pose corrections (local_solver.py:355-390)."""
        p, m = self.p, self.m
        nvv = verts.size
        s = p.cub_ids.shape[1]
        if s == 0:
            return np.zeros((nvv, 3, 3))
        ids, valid = p.cub_ids[verts], p.cub_valid[verts]
        uniq = np.unique(ids[valid]) if np.any(valid) else np.zeros(0, np.int64)
        if uniq.size == 0:
            return np.zeros((nvv, 3, 3))
        _, _, hc = element_terms(x[m.tets[uniq]], m.dm_inv[uniq], m.volumes[uniq],
                                 m.mu[uniq], m.lam[uniq], project=True)
        where = np.zeros(m.num_elements, dtype=np.int64)
        where[uniq] = np.arange(uniq.size)
        rw = rot[p.cub_verts[verts]]                                 # (v,s,4,3,3)
        ri = np.broadcast_to(rot[verts][:, None], rw.shape[:2] + (3, 3))
        rows = np.einsum("vskab,vskbc,vsdc->vskad", rw, p.cub_rows[verts], ri)
        rows = rows.reshape(nvv, s, 12, 3)
        hr = self.h_rest[ids].reshape(nvv, s, 4, 3, 4, 3)
        hrot = np.einsum("vskab,vskbmc,vsmdc->vskamd", rw, hr, rw).reshape(nvv, s, 12, 12)
        delta = hc[where[ids]] - hrot
        return np.einsum("vs,vsia,vsij,vsjb->vab", p.cub_w[verts] * valid, rows, delta, rows)

    def pair_rows(self, pairs, k, v, rot):
        """Coupling rows of pair k for sub-problem v (local_solver.py:85-112)."""
        if pairs.kind[k] == PLANE:
            return np.eye(3)
        rows = np.zeros((12, 3))
        tri = pairs.tri[k]
        bary = pairs.bary[k]
        if v == pairs.vertex[k]:
            rows[0:3] = np.eye(3)
            for j in range(3):
                rows[3 + 3 * j:6 + 3 * j] = bary[j] * np.eye(3)
            return rows
        j = int(np.flatnonzero(tri == v)[0])
        rows[3 + 3 * j:6 + 3 * j] = np.eye(3)
        rows[0:3] = bary[j] * np.eye(3)
        vr = self.p.vrows.get(int(v))
        if vr is not None:
            for c in range(3):
                w = int(tri[c])
                if c != j and w in vr:
                    rows[3 + 3 * c:6 + 3 * c] = rot[w] @ vr[w] @ rot[v].T
        return rows

    def add_pair_terms(self, x, verts, a, g, pairs, rot):
        """Contact rows into (A, g), own force already collected
        (local_solver.py:418-447, own_in_field=False)."""
        if not len(pairs):
            return
        slot = {int(v): k for k, v in enumerate(verts)}
        for k in range(len(pairs)):
            members = pairs.stencil(k)
            hit = [(int(mv), slot[int(mv)]) for mv in members if int(mv) in slot]
            if not hit:
                continue
            _, gp, hp = pair_terms(self.m, x, pairs, k, project=True)
            for v, kk in hit:
                rows = self.pair_rows(pairs, k, v, rot)
                a[kk] += rows.T @ hp @ rows
                if pairs.kind[k] == PLANE:
                    own = gp
                else:
                    pos = 0 if v == pairs.vertex[k] else 1 + int(np.flatnonzero(pairs.tri[k] == v)[0])
                    own = gp[3 * pos:3 * pos + 3]
                g[kk] += rows.T @ gp - own

    def reduced_systems(self, x, z, h, verts, g_asm, pairs, rot, q=None, corr=None):
        """Frozen Schur block + sampled correction (local_solver.py:392-416);
        q / corr given: the sweep-start collect and corrections (GS colours)."""
        p, m = self.p, self.m
        ri = rot[verts]
        a = -np.einsum("vab,vbc,vdc->vad", ri, p.gbar[verts], ri)
        if q is None:
            q = self.collect(rot, g_asm)
        qg = q[p.group[verts]].reshape(verts.size, -1)
        g = -np.einsum("vab,vbk,vk->va", ri, p.gbar_rows[verts], qg)
        a = a + (self.corrections(x, verts, rot) if corr is None else corr)
        a = 0.5 * (a + np.swapaxes(a, 1, 2))
        wmin = np.linalg.eigvalsh(a).min(axis=1)
        bad = wmin <= 0.0
        if np.any(bad):
            a[bad] += (1e-9 * m.masses[verts[bad]] / h ** 2 - wmin[bad])[:, None, None] * np.eye(3)
        self.add_pair_terms(x, verts, a, g, pairs, rot)
        return a, g

    @staticmethod
    def solve3(a, b):
        """Batched gesv with the scalar fallback (local_solver.py:72-82, 580-588)."""
        def one(ak, bk):
            try:
                d = np.linalg.solve(ak, bk)
                if np.all(np.isfinite(d)):
                    return d
            except np.linalg.LinAlgError:
                pass
            tr = np.trace(ak)
            return bk * (3.0 / tr) if tr > 0 else np.zeros(3)
        try:
            d = np.linalg.solve(a, b[..., None])[..., 0]
        except np.linalg.LinAlgError:
            d = np.stack([one(a[k], b[k]) for k in range(a.shape[0])])
        for k in np.flatnonzero(~np.all(np.isfinite(d), axis=1)):
            d[k] = one(a[k], b[k])
        return d

    def alpha_caps(self, x, verts, delta, pairs):
        """local_solver.py:450-470."""
        alpha = np.ones(verts.size)
        if not len(pairs):
            return alpha
        slot = {int(v): k for k, v in enumerate(verts)}
        dn = np.linalg.norm(delta, axis=1)
        for k in range(len(pairs)):
            d = pair_live_distance(self.m, x, pairs, k)
            for v in pairs.stencil(k):
                kk = slot.get(int(v))
                if kk is None:
                    continue
                if pairs.kind[k] == PLANE:
                    rate = max(-(delta[kk] @ self.m.planes[pairs.plane[k]].normal), 0.0)
                else:
                    rate = 2.0 * dn[kk]
                if rate > 0:
                    alpha[kk] = min(alpha[kk], 0.9 * d / rate)
        return np.minimum(alpha, 1.0)

    def line_search(self, x, verts, delta, pairs, a, g):
        """Quadratic-model local search (local_solver.py:523-553)."""
        cfg = self.cfg
        if not cfg.local_line_search:
            return np.ones(verts.size), 0
        alpha = self.alpha_caps(x, verts, delta, pairs)

        def model_at(al):
            st = al[:, None] * delta
            return np.einsum("vc,vc->v", st, g) + 0.5 * np.einsum("va,vab,vb->v", st, a, st)

        base = model_at(np.zeros(verts.size))
        acts = 0
        ok = np.zeros(verts.size, dtype=bool)
        for it in range(cfg.max_halvings + 1):
            ok |= model_at(alpha) <= base + 1e-12 * np.abs(base)
            if it == 0:
                acts = int(np.count_nonzero(~ok))
            if ok.all():
                break
            alpha[~ok] *= 0.5
            if alpha[~ok].max(initial=0.0) < cfg.alpha_floor:
                alpha[~ok] = cfg.alpha_floor
                break
        return alpha, acts

    def backtrack(self, z, h, x0, dx, e0, pairs):
        """Sweep-level guard (local_solver.py:555-577)."""
        m = self.m
        gamma = feasibility_cap(m, x0, dx) if (len(pairs) or m.planes) else 1.0
        halv = 0
        self.last_trial_energy = None
        while halv <= self.cfg.max_halvings:
            xt = x0 + gamma * dx
            try:
                et = total_energy(m, z, h, xt, find_pairs(m, xt))
            except Infeasible:
                et = np.inf
            if et <= e0 + 1e-12 * abs(e0):
                self.last_trial_energy = et
                break
            gamma *= 0.5
            halv += 1
        return x0 + gamma * dx, gamma * dx, halv

    def sweep(self, state, rot):
        """One outer iteration (Jacobi or Gauss-Seidel); mutates state.x
        (local_solver.py:606-655)."""
        m, p = self.m, self.p
        x, z, h = state.x, state.z, state.h
        pairs = find_pairs(m, x)
        info = {"line_search_activations": 0, "max_local_step": 0.0,
                "grad_norm": 0.0, "grad_sq": 0.0}
        guard = self.cfg.local_line_search
        e0 = total_energy(m, z, h, x, pairs) if guard else None
        verts = p.free
        dx = np.zeros_like(x)
        if self.cfg.mode == "jacobi":
            g_asm = self.assembled_field(x, z, h, pairs)
            a, g = self.reduced_systems(x, z, h, verts, g_asm, pairs, rot)
            delta = self.solve3(a, -g)
            alpha, acts = self.line_search(x, verts, delta, pairs, a, g)
            info["line_search_activations"] += acts
            info["grad_sq"] += float(np.sum(g_asm[~np.asarray(m.fixed_mask)] ** 2))
            dx[verts] = alpha[:, None] * delta
            state.x = x + dx
        else:
            # Gauss-Seidel (local_solver.py:627-649): collect and corrections
            # at the sweep start; per colour (ascending) pairs, assembled field,
            # reduced systems and local search at the current positions
            x_cur = x.copy()
            q0 = self.collect(rot, self.assembled_field(x, z, h, pairs))
            groups = self.color_groups()
            corr0 = [self.corrections(x, cv, rot) for cv in groups]
            for cv, c0 in zip(groups, corr0):
                cpairs = find_pairs(m, x_cur)
                g_asm = self.assembled_field(x_cur, z, h, cpairs)
                a, g = self.reduced_systems(x_cur, z, h, cv, g_asm, cpairs, rot, q=q0, corr=c0)
                delta = self.solve3(a, -g)
                alpha, acts = self.line_search(x_cur, cv, delta, cpairs, a, g)
                info["line_search_activations"] += acts
                info["grad_sq"] += float(np.sum(g_asm[cv] ** 2))
                step = alpha[:, None] * delta
                x_cur[cv] += step
                dx[cv] += step
            state.x = x_cur
        info["grad_norm"] = np.sqrt(info["grad_sq"])
        self.pairs = pairs
        if guard:
            state.x, dx, halv = self.backtrack(z, h, x, dx, e0, pairs)
            info["line_search_activations"] += halv
        info["max_local_step"] = float(np.linalg.norm(dx, axis=1).max(initial=0.0))
        return dx, info

    def color_groups(self):
        """Free vertices per colour, colours ascending (local_solver.py:298-303)."""
        colors = np.asarray(self.m.colors)
        free = ~np.asarray(self.m.fixed_mask)
        ncol = int(colors.max()) + 1 if colors.size else 0
        out = [np.flatnonzero((colors == c) & free) for c in range(ncol)]
        return [g for g in out if g.size]

    def outer_solve(self, state):
        """local_solver.py:688-721."""
        cfg, m = self.cfg, self.m
        st = OracleStats()
        t0 = time.perf_counter()
        for _ in range(cfg.max_outer):
            t1 = time.perf_counter()
            rot = vertex_rotations(m, state.x)
            state.rotations = rot
            dx, info = self.sweep(state, rot)
            st.wall_ms.append(1e3 * (time.perf_counter() - t1))
            dxn = float(m.normalization.scale * np.linalg.norm(dx))
            st.dx_norms.append(dxn)
            st.grad_norms.append(info["grad_norm"])
            st.max_local_steps.append(info["max_local_step"])
            st.line_search_activations.append(info["line_search_activations"])
            if cfg.track_energy:
                st.energies.append(total_energy(m, state.z, state.h, state.x,
                                                find_pairs(m, state.x)))
            st.outer_iterations += 1
            if dxn < cfg.tol_dx:
                st.converged = True
                break
        st.wall_seconds = time.perf_counter() - t0
        return st


# ============================================================ frame driver
def compute_z(model, x_prev, v, h):
    """z = x_prev + h v + h^2 g, fixed vertices pinned (assembly.py:165-180)."""
    z = x_prev + h * v + h * h * np.broadcast_to(model.gravity, x_prev.shape)
    fm = np.asarray(model.fixed_mask)
    z[fm] = x_prev[fm]
    return z


def initial_guess(model, x_prev, z):
    """Predictor warm start, feasibility-capped (harness.py:130-134)."""
    dx = z - x_prev
    return x_prev + feasibility_cap(model, x_prev, dx) * dx
