"""The reference's on-disk formats either side of the hot path (SURVEY §8(f)
rank 4), so ``tetsolve run`` outputs and precompute caches carry over:

* ``metrics.csv``: per-sweep solver statistics (harness.py:21-22, 137-155);
* per-frame surface ``.obj`` and ``.node``/``.ele`` state dumps
  (mesh.py:284-307, written by harness.run, harness.py:203-211);
* the precompute caches, i.e. per-vertex bases and cubature sets as ``.npz``
  (subspace.py:282-312, cubature.py:327-346). They load into a
  :class:`Precompute`, so a cache the reference trained can drive the GPU
  path directly.

``run_frames`` is the harness.run time-stepping loop (harness.py:160-219)
around any solver with ``outer_solve(state)``, writing the same files.
Formats are byte-identical to the reference's writers
(tests/test_formats.py against fixtures the reference wrote).
"""

import csv
from pathlib import Path

import numpy as np

from .model import compute_z, step_velocity_update
from .precompute import Precompute

METRICS_HEADER = ("frame", "iter", "solver", "energy", "dx_norm", "grad_norm", "wall_ms")


def stats_rows(frame, tag, stats):
    """Rows of one frame's IterationStats (harness.py:148-157)."""
    rows = []
    for k in range(len(stats.dx_norms)):
        energy = stats.energies[k] if k < len(stats.energies) else np.nan
        wall = stats.wall_ms[k] if k < len(stats.wall_ms) else 0.0
        rows.append((frame, k, tag, energy, stats.dx_norms[k], stats.grad_norms[k], wall))
    return rows


def write_metrics(path, rows):
    """metrics.csv (harness.py:137-145): 17 significant digits, wall_ms 6."""
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(METRICS_HEADER)
        for r in rows:
            w.writerow([r[0], r[1], r[2], f"{r[3]:.17g}", f"{r[4]:.17g}", f"{r[5]:.17g}", f"{r[6]:.6g}"])


def read_metrics(path):
    """metrics.csv rows as (frame, iter, solver, energy, dx_norm, grad_norm, wall_ms)."""
    with open(path, newline="") as fh:
        r = csv.reader(fh)
        head = tuple(next(r))
        if head != METRICS_HEADER:
            raise ValueError(f"{path}: not a metrics.csv header: {head}")
        return [(int(a), int(b), c, float(d), float(e), float(f), float(g)) for a, b, c, d, e, f, g in r]


def export_obj(path, positions, surface_tris):
    """Surface as Wavefront OBJ, 1-based faces, 9 significant digits (mesh.py:302-307)."""
    p = np.asarray(positions, dtype=np.float64)
    t = np.asarray(surface_tris, dtype=np.int64) + 1
    with open(path, "w") as fh:
        fh.write("".join(f"v {a:.9g} {b:.9g} {c:.9g}\n" for a, b, c in p))
        fh.write("".join(f"f {a} {b} {c}\n" for a, b, c in t))


def save_mesh(tets, positions, node_path, ele_path):
    """.node/.ele text, 0-based ids, 17 significant digits (mesh.py:284-299)."""
    pos = np.asarray(positions, dtype=np.float64)
    tets = np.asarray(tets, dtype=np.int64)
    with open(node_path, "w") as fh:
        fh.write(f"{pos.shape[0]} 3 0 0\n")
        fh.write("".join(f"{j} {p[0]:.17g} {p[1]:.17g} {p[2]:.17g}\n" for j, p in enumerate(pos)))
    with open(ele_path, "w") as fh:
        fh.write(f"{tets.shape[0]} 4 0\n")
        fh.write("".join(f"{e} {t[0]} {t[1]} {t[2]} {t[3]}\n" for e, t in enumerate(tets)))


def load_precompute_cache(bases_path, cubature_path):
    """A Precompute from the reference's cache files (subspace.save_bases /
    cubature.save_cubature layouts, subspace.py:282-299, cubature.py:327-335).
    Returns (precompute, info) with info = {"h_ref", "mode"}."""
    b = np.load(bases_path, allow_pickle=False)
    c = np.load(cubature_path, allow_pickle=False)
    verts = np.asarray(b["vertices"], dtype=np.int64)
    glen = [b[f"group_{v}"].size for v in verts]
    gmax = max(glen, default=1)
    group = np.full((verts.size, gmax), -1, dtype=np.int64)
    grows = np.zeros((verts.size, 3, 3 * gmax))
    keys, ptr, blocks, cptr, ce, cw = [], [0], [], [0], [], []
    for k, v in enumerate(verts):
        group[k, :glen[k]] = b[f"group_{v}"]
        grows[k, :, :3 * glen[k]] = b[f"grows_{v}"]
        rk = np.asarray(b[f"rkeys_{v}"], dtype=np.int64)
        keys.extend(rk.tolist())
        blocks.append(np.asarray(b[f"rows_{v}"]).reshape(-1, 3, 3))
        ptr.append(len(keys))
        ce.extend(np.asarray(c[f"elems_{v}"], dtype=np.int64).tolist())
        cw.extend(np.asarray(c[f"weights_{v}"], dtype=np.float64).tolist())
        cptr.append(len(ce))
    pre = Precompute(vertices=verts, gbar=np.stack([b[f"gbar_{v}"] for v in verts]),
                     group=group, gbar_rows=grows,
                     vrows_ptr=np.array(ptr, dtype=np.int64),
                     vrows_keys=np.array(keys, dtype=np.int64),
                     vrows=np.concatenate(blocks) if blocks else np.zeros((0, 3, 3)),
                     cub_ptr=np.array(cptr, dtype=np.int64),
                     cub_elems=np.array(ce, dtype=np.int64),
                     cub_weights=np.array(cw, dtype=np.float64))
    info = {"h_ref": float(b["h_ref"][0]), "mode": str(b["mode"][0])}
    return pre, info


def run_frames(model, solver, state, frames, out_dir, tag="jgs2_cubature", dumps=True):
    """harness.run's loop (harness.py:186-219) around ``solver.outer_solve``:
    compute_z, capped initialize_step, outer_solve, velocity update, then the
    per-frame .obj and per-body .node/.ele dumps and metrics.csv. Returns the
    list of frames that did not converge."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    rows, failed = [], []
    offsets = list(getattr(model, "bodies", [])) or [0]
    for frame in range(1, frames + 1):
        compute_z(model, state)
        solver.initialize_step(state)
        stats = solver.outer_solve(state)
        rows.extend(stats_rows(frame, tag, stats))
        if not stats.converged:
            failed.append(frame)
        step_velocity_update(model, state, state.x)
        if dumps:
            export_obj(out / f"frame_{frame:04d}.obj", state.x, model.surface_tris)
            _dump_bodies(model, state.x, out, frame)
    write_metrics(out / "metrics.csv", rows)
    return failed


def _dump_bodies(model, x, out, frame):
    vb = np.asarray(model.vertex_body)
    tb = np.asarray(model.tet_body)
    for bi in range(int(vb.max()) + 1 if vb.size else 0):
        vs = np.flatnonzero(vb == bi)
        tets = np.asarray(model.tets)[tb == bi] - vs[0]
        save_mesh(tets, x[vs], out / f"body{bi}_frame_{frame:04d}.node",
                  out / f"body{bi}_frame_{frame:04d}.ele")
