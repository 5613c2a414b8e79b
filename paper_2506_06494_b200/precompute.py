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
    def injected(cls, model, h_ref, samples=6, seed=0, weight_scale=0.05):
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
        rng = np.random.default_rng(seed)
        nv, ne = model.num_vertices, model.num_elements
        tets = np.asarray(model.tets)
        free = np.flatnonzero(~np.asarray(model.fixed_mask))
        diag = rest_diagonal_blocks(model, h_ref)
        ptr_inc = np.zeros(nv + 1, dtype=np.int64)
        np.cumsum(np.bincount(tets.ravel(), minlength=nv), out=ptr_inc[1:])
        inc = np.argsort(tets.ravel(), kind="stable") // 4
        tb = np.asarray(getattr(model, "tet_body", np.zeros(ne, dtype=np.int64)))
        body_lo = np.zeros(ne, dtype=np.int64)
        body_hi = np.zeros(ne, dtype=np.int64)
        for b in np.unique(tb):
            idx = np.flatnonzero(tb == b)
            body_lo[idx] = idx.min()
            body_hi[idx] = idx.max() + 1
        # Cubature samples: element ids near an incident element, rejecting
        # incident ones (retry by shifting).
        first_inc = inc[ptr_inc[free]]
        off = rng.integers(24, 4000, size=(free.size, samples)) * \
            rng.choice((-1, 1), size=(free.size, samples))
        cand = first_inc[:, None] + off
        lo = body_lo[first_inc][:, None]
        hi = body_hi[first_inc][:, None]
        span = np.maximum(hi - lo, 1)
        cand = lo + np.mod(cand - lo, span)
        cub = np.sort(cand, axis=1)
        # drop duplicates / incident collisions by nudging (rare)
        for c in range(1, samples):
            dup = cub[:, c] <= cub[:, c - 1]
            cub[dup, c] = np.minimum(cub[dup, c - 1] + 1, hi[dup, 0] - 1)
        inc_sets = [set(inc[ptr_inc[v]:ptr_inc[v + 1]].tolist()) for v in free] \
            if free.size <= 200000 else None
        weights = weight_scale * rng.uniform(0.5, 1.5, size=cub.shape)
        # Retained rows: own, incident-element vertices, cubature vertices.
        x0 = np.asarray(model.rest_positions)
        ext = float(np.ptp(x0, axis=0).max()) or 1.0
        keys_list, ptr = [], [0]
        for k, v in enumerate(free):
            kk = set(tets[inc[ptr_inc[v]:ptr_inc[v + 1]]].ravel().tolist())
            kk.add(int(v))
            elems = cub[k]
            if inc_sets is not None:
                bad = [e for e in elems if e in inc_sets[k]]
                if bad:
                    keep = [e for e in elems if e not in inc_sets[k]]
                    elems = np.array(keep, dtype=np.int64)
                    weights_k = weights[k][:len(keep)]
                    cub[k, :len(keep)] = elems
                    cub[k, len(keep):] = -1
                    weights[k, :len(keep)] = weights_k
                    weights[k, len(keep):] = 0.0
            kk.update(tets[elems[elems >= 0]].ravel().tolist())
            keys_list.append(np.array(sorted(kk), dtype=np.int64))
            ptr.append(ptr[-1] + len(kk))
        keys = np.concatenate(keys_list) if keys_list else np.zeros(0, np.int64)
        owner = np.repeat(free, np.diff(ptr))
        dist = np.linalg.norm(x0[keys] - x0[owner], axis=1) / ext
        scale = np.where(keys == owner, 1.0, 0.6 * np.exp(-8.0 * dist))
        vrows = scale[:, None, None] * np.eye(3)[None]
        valid = cub >= 0
        cptr = np.zeros(free.size + 1, dtype=np.int64)
        np.cumsum(valid.sum(axis=1), out=cptr[1:])
        return cls(vertices=free.astype(np.int64), gbar=-diag[free],
                   group=free[:, None].astype(np.int64), gbar_rows=-diag[free],
                   vrows_ptr=np.array(ptr, dtype=np.int64), vrows_keys=keys,
                   vrows=vrows, cub_ptr=cptr, cub_elems=cub[valid].astype(np.int64),
                   cub_weights=weights[valid])


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
