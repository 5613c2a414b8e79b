"""Precompute inputs of the runtime path: per-vertex bases and cubature sets.

The reference produces these in ``harness.prepare`` (``harness.py:57-107``)
as ``{vertex: PerturbationBasis}`` (``subspace.py:33-45``) and
``{vertex: CubatureSet}`` (``cubature.py:22-27``). ``Precompute`` is the flat
(CSR) form both the CUDA path and the oracle consume. Constructors:

* ``from_reference(bases, sets)`` -- the reference's own dicts (drop-in);
* ``from_arrays(npz)`` -- the golden-fixture layout (``tests/golden``);
* ``injected(model, h_ref, ...)`` -- structurally valid synthetic precompute
  for benchmark scales where the reference precompute (dense N x 3 basis per
  vertex, ``subspace.py:155-183``) cannot run.
  Iteration counts under injected inputs are not reference-comparable;
  per-sweep throughput is.
"""

from dataclasses import dataclass

import numpy as np

KEYS = ("vertices", "gbar", "group", "gbar_rows", "vrows_ptr", "vrows_keys",
        "vrows", "cub_ptr", "cub_elems", "cub_weights")


@dataclass
class Precompute:
    vertices: np.ndarray    # (nb,) sorted free vertex ids with a basis
    gbar: np.ndarray        # (nb, 3, 3)
    group: np.ndarray       # (nb, gmax) -1 padded
    gbar_rows: np.ndarray   # (nb, 3, 3*gmax)
    vrows_ptr: np.ndarray   # (nb+1,)
    vrows_keys: np.ndarray  # retained vertex ids, ascending per basis
    vrows: np.ndarray       # (nnz, 3, 3)
    cub_ptr: np.ndarray     # (nb+1,)
    cub_elems: np.ndarray
    cub_weights: np.ndarray

    def __getitem__(self, key):
        return getattr(self, key)

    @classmethod
    def from_arrays(cls, arrays, prefix="pre_"):
        return cls(**{k: np.asarray(arrays[prefix + k]) for k in KEYS})

    @classmethod
    def from_reference(cls, bases, sets):
        verts = np.array(sorted(bases), dtype=np.int64)
        glen = [len(bases[v].group) for v in verts]
        gmax = max(glen, default=1)
        group = np.full((verts.size, gmax), -1, dtype=np.int64)
        grows = np.zeros((verts.size, 3, 3 * gmax))
        keys, ptr, blocks, cptr, ce, cw = [], [0], [], [0], [], []
        for k, v in enumerate(verts):
            b = bases[v]
            group[k, :glen[k]] = b.group
            grows[k, :, :3 * glen[k]] = b.gbar_rows
            kk = sorted(b.vrows)
            keys.extend(kk)
            blocks.extend(b.vrows[w] for w in kk)
            ptr.append(len(keys))
            s = sets[v]
            ce.extend(int(e) for e in s.elements)
            cw.extend(float(w) for w in s.weights)
            cptr.append(len(ce))
        return cls(vertices=verts, gbar=np.stack([bases[v].gbar for v in verts]),
                   group=group, gbar_rows=grows,
                   vrows_ptr=np.array(ptr, dtype=np.int64),
                   vrows_keys=np.array(keys, dtype=np.int64),
                   vrows=np.array(blocks, dtype=np.float64).reshape(-1, 3, 3),
                   cub_ptr=np.array(cptr, dtype=np.int64),
                   cub_elems=np.array(ce, dtype=np.int64),
                   cub_weights=np.array(cw, dtype=np.float64))

    @classmethod
    def injected(cls, model, h_ref, samples=6, seed=0, weight_scale=0.05, neighbor_scale=0.6):
        """Structurally valid synthetic precompute (bench scales only).

        * Gbar_v = -Hbar_vv (the vertex's own rest block, elastic + inertia):
          with zero correction the local step is then exactly the co-rotated
          rest-Newton step -R_i q_i (any SPD -Gbar gives it), so sweeps
          converge like the real method.
        * ``samples`` cubature elements per vertex drawn from the same body,
          not incident to the vertex, biased to its neighbourhood (random
          offsets in element id space), with small weights.
        * Retained rows: identity at the vertex, a distance-decayed multiple
          of the identity at incident/cubature vertices (the shape of a true
          perturbation basis, which decays away from the vertex).
        """
        import scipy.sparse as sp
        rng = np.random.default_rng(seed)
        nv, ne = model.num_vertices, model.num_elements
        tets = np.asarray(model.tets, dtype=np.int64)
        free = np.flatnonzero(~np.asarray(model.fixed_mask))
        nf = free.size
        diag = rest_diagonal_blocks_chunked(model, h_ref)
        flat = tets.ravel()
        eid = np.repeat(np.arange(ne, dtype=np.int64), 4)
        ptr_inc = np.zeros(nv + 1, dtype=np.int64)
        np.cumsum(np.bincount(flat, minlength=nv), out=ptr_inc[1:])
        inc = eid[np.argsort(flat, kind="stable")]
        tb = np.asarray(getattr(model, "tet_body", np.zeros(ne, dtype=np.int64)))
        starts = np.flatnonzero(np.r_[True, tb[1:] != tb[:-1]])
        ends = np.r_[starts[1:], ne]
        seg = np.searchsorted(starts, np.arange(ne), side="right") - 1
        body_lo, body_hi = starts[seg], ends[seg]
        has_inc = ptr_inc[free + 1] > ptr_inc[free]
        first_inc = np.where(has_inc, inc[np.minimum(ptr_inc[free], max(inc.size - 1, 0))], 0)
        # cubature samples: element ids at random offsets from an incident
        # element (same body), sorted, de-duplicated, never incident
        off = rng.integers(24, 4000, size=(nf, samples)) * rng.choice((-1, 1), size=(nf, samples))
        lo = body_lo[first_inc][:, None]
        span = np.maximum(body_hi[first_inc][:, None] - lo, 1)
        cub = np.sort(lo + np.mod(first_inc[:, None] + off - lo, span), axis=1)
        dup = np.zeros_like(cub, dtype=bool)
        dup[:, 1:] = cub[:, 1:] == cub[:, :-1]
        inc_key = np.sort(flat * ne + eid) if ne else np.zeros(0, np.int64)
        q = free[:, None] * ne + cub
        pos = np.searchsorted(inc_key, q)
        is_inc = (pos < inc_key.size) & (inc_key[np.minimum(pos, inc_key.size - 1)] == q)
        valid = ~(dup | is_inc | ~has_inc[:, None])
        weights = weight_scale * rng.uniform(0.5, 1.5, size=cub.shape)
        # retained rows: own + incident-element vertices + cubature corners
        A = sp.csr_matrix((np.ones(flat.size, dtype=np.int8), (flat, eid)), shape=(nv, max(ne, 1)))
        adj = (A @ A.T)[free]
        rows_c = np.repeat(np.arange(nf), 4 * samples)
        cols_c = tets[np.where(valid, cub, 0)].reshape(nf, -1)
        keep_c = np.repeat(valid, 4, axis=1).ravel()
        Pc = sp.csr_matrix((np.ones(int(keep_c.sum()), dtype=np.int8),
                            (rows_c[keep_c], cols_c.ravel()[keep_c])), shape=(nf, nv))
        I = sp.csr_matrix((np.ones(nf, dtype=np.int8), (np.arange(nf), free)), shape=(nf, nv))
        K = (adj.astype(bool) + Pc.astype(bool) + I.astype(bool)).tocsr()
        K.sort_indices()
        keys = K.indices.astype(np.int64)
        ptr = K.indptr.astype(np.int64)
        owner = np.repeat(free, np.diff(ptr))
        x0 = np.asarray(model.rest_positions)
        ext = float(np.ptp(x0, axis=0).max()) or 1.0
        dist = np.linalg.norm(x0[keys] - x0[owner], axis=1) / ext
        scale = np.where(keys == owner, 1.0, neighbor_scale * np.exp(-8.0 * dist))
        vrows = np.zeros((keys.size, 3, 3))
        vrows[:, 0, 0] = vrows[:, 1, 1] = vrows[:, 2, 2] = scale
        cptr = np.zeros(nf + 1, dtype=np.int64)
        np.cumsum(valid.sum(axis=1), out=cptr[1:])
        return cls(vertices=free.astype(np.int64), gbar=-diag[free],
                   group=free[:, None].astype(np.int64), gbar_rows=-diag[free],
                   vrows_ptr=ptr, vrows_keys=keys, vrows=vrows, cub_ptr=cptr,
                   cub_elems=cub[valid].astype(np.int64), cub_weights=weights[valid])


def rest_diagonal_blocks(model, h_ref):
    """Own 3x3 blocks of the rest Hessian M/h^2 + sum_e V W^T H9(I) W.

    At F = I the stable Neo-Hookean H9 is PSD, so the projected and
    unprojected element Hessians agree to rounding.
    H9(I) = mu_s*(1-1/4) I9 + 2 mu_s/16 f f^T + lam_s g g^T + s*skew, with
    f = g = vec(I), s = lam_s*(1-alpha)  (energy.py:110-141 at F = I).
    """
    tets = np.asarray(model.tets)
    nv = model.num_vertices
    mu = np.asarray(model.mu)
    lam = np.asarray(model.lam)
    mu_s = 4.0 * mu / 3.0
    lam_s = lam + 5.0 * mu / 6.0
    alpha = 1.0 + 0.75 * mu_s / lam_s
    dm_inv = np.asarray(model.dm_inv)
    W = np.empty(dm_inv.shape[:-2] + (4, 3))
    W[:, 1:, :] = dm_inv
    W[:, 0, :] = -dm_inv.sum(axis=-2)
    out = np.zeros((nv, 3, 3))
    out += (np.asarray(model.masses) / h_ref ** 2)[:, None, None] * np.eye(3)
    vol = np.asarray(model.volumes)
    # Diagonal block m of H12: V * sum_{j,k} W[m,j] W[m,k] H9[(j,r),(k,s)].
    # H9 at F=I, blocks (j,k) 3x3: c1*delta_jk I + c2 e_j e_k^T + c3 e_j e_k^T
    # ... computed generically below (small, vectorised over elements).
    eye = np.eye(3)
    fv = eye.T.reshape(9)  # vec(I)
    H9 = (mu_s * 0.75)[:, None, None] * np.eye(9)[None]
    H9 = H9 + (2.0 * mu_s / 16.0)[:, None, None] * np.outer(fv, fv)[None]
    H9 = H9 + lam_s[:, None, None] * np.outer(fv, fv)[None]
    s = lam_s * (1.0 - alpha)
    skew = np.zeros((9, 9))

    def sk(v):
        return np.array([[0, -v[2], v[1]], [v[2], 0, -v[0]], [-v[1], v[0], 0]])
    e = eye
    for bi, bj, blk in ((0, 1, -sk(e[2])), (0, 2, sk(e[1])), (1, 0, sk(e[2])),
                        (1, 2, -sk(e[0])), (2, 0, -sk(e[1])), (2, 1, sk(e[0]))):
        skew[3 * bi:3 * bi + 3, 3 * bj:3 * bj + 3] = blk
    H9 = H9 + s[:, None, None] * skew[None]
    H9b = H9.reshape(-1, 3, 3, 3, 3)  # [j, r, k, s]
    for m in range(4):
        blk = np.einsum("ej,ejrks,ek->ers", W[:, m], H9b, W[:, m]) * vol[:, None, None]
        np.add.at(out, tets[:, m], blk)
    return out


def rest_diagonal_blocks_chunked(model, h_ref, chunk=400000):
    """rest_diagonal_blocks over element chunks (bounded temporaries)."""
    class _View:
        pass
    ne = model.num_elements
    out = None
    for a in range(0, max(ne, 1), chunk):
        v = _View()
        sl = slice(a, min(ne, a + chunk))
        v.tets, v.mu, v.lam = np.asarray(model.tets)[sl], np.asarray(model.mu)[sl], np.asarray(model.lam)[sl]
        v.dm_inv, v.volumes = np.asarray(model.dm_inv)[sl], np.asarray(model.volumes)[sl]
        v.num_vertices = model.num_vertices
        v.masses = np.asarray(model.masses) if a == 0 else np.zeros(model.num_vertices)
        blk = rest_diagonal_blocks(v, h_ref)
        out = blk if out is None else out + blk
    return out
