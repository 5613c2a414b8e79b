"""Golden-trajectory replay shared by the oracle tests and the GPU parity tests."""

import numpy as np

from paper_2506_06494_b200.model import Model, SystemState
from paper_2506_06494_b200.precompute import Precompute

SCENES_SMALL = ("beam", "beam_stiff", "cube_drop", "two_body")
POS_RTOL = 1e-9  # north_star: FP64 positions within 1e-9 relative


def scene_inputs(g):
    """(model, precompute or None for plain-mode fixtures, h)."""
    model = Model.from_arrays(g)
    pre = Precompute.from_arrays(g) if "pre_vertices" in g else None
    h = float(g["scene_h"][0])
    return model, pre, h


def rel_err(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def pair_key(rows):
    """Bit-exact pair identity: (kind, vertex, tri, plane, bary zero pattern)."""
    out = []
    for r in rows:
        out.append((int(r[0]), int(r[1]), int(r[2]), int(r[3]), int(r[4]), int(r[5]),
                    tuple(bool(b != 0.0) for b in r[7:10])))
    return out


def replay(g, sweep_fn, pairs_fn, max_frames=None):
    """Drive every golden frame from the golden frame-start state.

    ``sweep_fn(state) -> (dx, info)`` runs one outer iteration (rotations
    refreshed inside, like ``outer_solve``); ``pairs_fn(x)`` returns the pair
    rows at x. Returns a report dict of worst errors and mismatches.
    """
    model, pre, h = scene_inputs(g)
    cfg = g["scene_cfg"]
    tol_dx, max_outer = float(cfg[0]), int(cfg[1])
    frames = g["frame_iterations"].size if max_frames is None else max_frames
    traj_f, traj_s = g["traj_frame"], g["traj_sweep"]
    ptr = g["pairs_ptr"]
    rep = {"pos": 0.0, "dxn": 0.0, "iters_ref": [], "iters": [], "pair_mismatch": 0,
           "sweeps": 0}
    row = 0
    for f in range(frames):
        state = SystemState(x=g["frame_x_init"][f].copy(), x_prev=g["frame_x_prev"][f].copy(),
                            v=g["frame_v"][f].copy(), z=g["frame_z"][f].copy(), h=h)
        n_ref = int(g["frame_iterations"][f])
        it = 0
        for it in range(1, max_outer + 1):
            if row < traj_f.size and traj_f[row] == f + 1 and traj_s[row] == it:
                ref_pairs = g["pairs"][ptr[row]:ptr[row + 1]]
                got = pairs_fn(state.x)
                if pair_key(got) != pair_key(ref_pairs):
                    rep["pair_mismatch"] += 1
            dx, info = sweep_fn(state)
            dxn = model.dx_norm(dx)
            if row < traj_f.size and traj_f[row] == f + 1 and traj_s[row] == it:
                rep["pos"] = max(rep["pos"], rel_err(state.x, g["traj_x"][row]))
                rep["dxn"] = max(rep["dxn"], abs(dxn - g["traj_dx_norm"][row])
                                 / max(g["traj_dx_norm"][row], 1e-300))
                rep["sweeps"] += 1
                row += 1
            if dxn < tol_dx:
                break
        while row < traj_f.size and traj_f[row] == f + 1:
            row += 1
        rep["iters_ref"].append(n_ref)
        rep["iters"].append(it)
    return rep


def reference_objects(pre):
    """The reference's precompute objects rebuilt from the flat fixture form:
    ``{vertex: PerturbationBasis}`` (subspace.py:33-45) and ``{vertex:
    CubatureSet}`` (cubature.py:22-27) -- the reference's own classes when
    ``tetsolve`` is importable, else namespaces with the same attributes (the
    drop-in reads them duck-typed, like the reference's LocalSolver)."""
    from types import SimpleNamespace
    try:
        from tetsolve.subspace import PerturbationBasis
        from tetsolve.cubature import CubatureSet
    except Exception:
        PerturbationBasis = CubatureSet = None
    bases, sets = {}, {}
    for k, v in enumerate(np.asarray(pre.vertices)):
        v = int(v)
        grp = np.asarray(pre.group[k])
        grp = grp[grp >= 0]
        lo, hi = int(pre.vrows_ptr[k]), int(pre.vrows_ptr[k + 1])
        vrows = {int(w): np.asarray(pre.vrows[j]) for j, w in zip(range(lo, hi), pre.vrows_keys[lo:hi])}
        kw = dict(vertex=v, gbar=np.asarray(pre.gbar[k]), vrows=vrows, reduced_mass=np.zeros((3, 3)),
                  group=grp, gbar_rows=np.asarray(pre.gbar_rows[k][:, :3 * grp.size]))
        bases[v] = PerturbationBasis(**kw) if PerturbationBasis else SimpleNamespace(**kw)
        c0, c1 = int(pre.cub_ptr[k]), int(pre.cub_ptr[k + 1])
        ckw = dict(elements=np.asarray(pre.cub_elems[c0:c1]), weights=np.asarray(pre.cub_weights[c0:c1]))
        sets[v] = CubatureSet(**ckw) if CubatureSet else SimpleNamespace(**ckw)
    return bases, sets
