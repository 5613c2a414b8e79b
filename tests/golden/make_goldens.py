"""Generate golden fixtures by running the REFERENCE package (tetsolve) here.

This script is the only place that imports the reference. It runs in the
build container (where /root/reference is mounted read-only) and writes small
``.npz`` fixtures under ``tests/golden/`` that travel to the GPU box; nothing at
test or bench time reads /root/reference.

Per scene it records:
  * the reference ``Model`` static arrays (so the product's model builder and
    the CUDA path consume byte-identical inputs),
  * the precompute (per-vertex bases + cubature sets) from ``harness.prepare``
    (``harness.py:57-107``),
  * a trajectory driven exactly like ``LocalSolver.outer_solve``
    (``local_solver.py:688-721``) but with per-sweep snapshots: positions,
    dx norms, grad norms, energies, activations, and the active contact-pair
    set at the start of every sweep (``local_solver.py:612``),
  * per-kernel intermediates at one mid-trajectory state via the reference's
    private methods (rotations, assembled field, collect, sampled corrections,
    reduced systems, batch solve, line search, total energy).

Usage (build container only):
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_goldens.py [scene ...]
"""

import os
import sys
import time
from pathlib import Path

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
os.environ.setdefault("TETSOLVE_CACHE_DIR", "/tmp/tetsolve_cache_goldens")

import numpy as np  # noqa: E402
import scipy  # noqa: E402

from tetsolve import harness, subspace, cubature  # noqa: E402
from tetsolve.assembly import (Model, SystemState, compute_z,  # noqa: E402
                               step_velocity_update, total_energy)
from tetsolve.energy import MaterialParams, BarrierParams  # noqa: E402
from tetsolve.local_solver import LocalSolver, SolverConfig  # noqa: E402
from tetsolve.primitives import box_grid  # noqa: E402
from tetsolve.scene import CubatureConfig, parse_scene  # noqa: E402

OUT = Path(__file__).resolve().parent


def model_arrays(model):
    d = {
        "rest_positions": model.rest_positions,
        "initial_positions": model.initial_positions,
        "tets": model.tets,
        "volumes": model.volumes,
        "dm_inv": model.dm_inv,
        "mu": model.mu,
        "lam": model.lam,
        "masses": model.masses,
        "elem_qmass": model.elem_qmass,
        "fixed_mask": model.fixed_mask,
        "colors": model.colors,
        "vertex_body": model.vertex_body,
        "tet_body": model.tet_body,
        "surface_tris": model.surface_tris,
        "surface_tri_body": model.surface_tri_body,
        "surface_vertices": model.surface_vertices,
        "gravity": model.gravity,
        "norm_scale": np.array([model.normalization.scale]),
        "plane_points": np.array([p.point for p in model.planes]).reshape(-1, 3),
        "plane_normals": np.array([p.normal for p in model.planes]).reshape(-1, 3),
        "barrier": np.array([model.barrier.dhat, model.barrier.kappa])
        if model.barrier is not None else np.zeros(0),
        "body_vertex_offsets": np.array([b.vertex_offset for b in model.bodies]),
        "body_element_offsets": np.array([b.element_offset for b in model.bodies]),
    }
    return {f"model_{k}": np.asarray(v) for k, v in d.items()}


def precompute_arrays(bases, sets):
    verts = np.array(sorted(bases), dtype=np.int64)
    gbar = np.stack([bases[v].gbar for v in verts])
    group_len = np.array([len(bases[v].group) for v in verts])
    gmax = int(group_len.max())
    group = np.full((verts.size, gmax), -1, dtype=np.int64)
    grows = np.zeros((verts.size, 3, 3 * gmax))
    for k, v in enumerate(verts):
        group[k, :group_len[k]] = bases[v].group
        grows[k, :, :3 * group_len[k]] = bases[v].gbar_rows
    rkeys, rptr, rblocks = [], [0], []
    for v in verts:
        keys = sorted(bases[v].vrows)
        rkeys.extend(keys)
        rblocks.extend(bases[v].vrows[w] for w in keys)
        rptr.append(len(rkeys))
    cptr, celems, cw, cres = [0], [], [], []
    for v in verts:
        s = sets[v]
        celems.extend(int(e) for e in s.elements)
        cw.extend(float(w) for w in s.weights)
        cptr.append(len(celems))
        cres.append(s.residual)
    return {
        "pre_vertices": verts,
        "pre_gbar": gbar,
        "pre_group": group,
        "pre_gbar_rows": grows,
        "pre_reduced_mass": np.stack([bases[v].reduced_mass for v in verts]),
        "pre_vrows_ptr": np.array(rptr, dtype=np.int64),
        "pre_vrows_keys": np.array(rkeys, dtype=np.int64),
        "pre_vrows": np.array(rblocks).reshape(-1, 3, 3),
        "pre_cub_ptr": np.array(cptr, dtype=np.int64),
        "pre_cub_elems": np.array(celems, dtype=np.int64),
        "pre_cub_weights": np.array(cw),
        "pre_cub_residual": np.array(cres),
    }


def pair_rows(pairs):
    """(kind, vertex, tri0..2, plane, d, bary0..2) rows; kind 0=plane 1=tri."""
    out = np.zeros((len(pairs), 10))
    for k, p in enumerate(pairs):
        out[k, 0] = 0 if p.kind == "plane" else 1
        out[k, 1] = p.vertex
        if p.kind != "plane":
            out[k, 2:5] = p.tri
            out[k, 7:10] = p.bary
        out[k, 5] = p.plane
        out[k, 6] = p.d
    return out


def run_trajectory(model, solver, h, frames, record_kernels_at=(2, 1)):
    """Drive frames exactly like harness.run (+outer_solve), with snapshots."""
    cfg = solver.config
    state = SystemState.initial(model, h)
    rec = {k: [] for k in ("frame", "sweep", "x", "dx_norm", "grad_norm",
                           "energy", "max_local_step", "activations")}
    frame_rec = {k: [] for k in ("x_prev", "v", "z", "x_init", "iterations",
                                 "converged", "x_final")}
    pair_log, pair_ptr = [], [0]
    kernels = {}
    for frame in range(1, frames + 1):
        compute_z(model, state)
        harness.initialize_step(model, state)
        frame_rec["x_prev"].append(state.x_prev.copy())
        frame_rec["v"].append(state.v.copy())
        frame_rec["z"].append(state.z.copy())
        frame_rec["x_init"].append(state.x.copy())
        converged = False
        it = 0
        for it in range(1, cfg.max_outer + 1):
            rot = subspace.vertex_rotations(model, state.x)
            state.rotations = rot
            pairs = model.find_pairs(state.x)
            pair_log.append(pair_rows(pairs))
            pair_ptr.append(pair_ptr[-1] + len(pairs))
            if (frame, it) == tuple(record_kernels_at):
                kernels = kernel_snapshot(model, solver, state, rot, pairs)
            dx, info = solver.sweep(state, rotations=rot)
            dxn = model.dx_norm(dx)
            e = total_energy(model, state, state.x, model.find_pairs(state.x))
            rec["frame"].append(frame)
            rec["sweep"].append(it)
            rec["x"].append(state.x.copy())
            rec["dx_norm"].append(dxn)
            rec["grad_norm"].append(info["grad_norm"])
            rec["energy"].append(e)
            rec["max_local_step"].append(info["max_local_step"])
            rec["activations"].append(info["line_search_activations"])
            if dxn < cfg.tol_dx:
                converged = True
                break
        frame_rec["iterations"].append(it)
        frame_rec["converged"].append(converged)
        frame_rec["x_final"].append(state.x.copy())
        step_velocity_update(model, state, state.x)
    out = {f"traj_{k}": np.asarray(v) for k, v in rec.items()}
    out.update({f"frame_{k}": np.asarray(v) for k, v in frame_rec.items()})
    out["pairs"] = np.concatenate(pair_log) if pair_log else np.zeros((0, 10))
    out["pairs_ptr"] = np.array(pair_ptr, dtype=np.int64)
    out.update(kernels)
    return out


def kernel_snapshot(model, solver, state, rot, pairs):
    """Per-kernel intermediates from the reference's private methods."""
    x = state.x.copy()
    verts = solver.free
    if solver.config.subspace == "none":  # plain VBD (local_solver.py:325-353, 472-522)
        g_asm = solver._assembled_field(x, state, pairs)
        a, g = solver._plain_systems(x, state, verts, g_asm, pairs, rot)
        delta = solver._solve_batch(a, -g)
        alpha, acts = solver._line_search(x, state, verts, delta, pairs, rot, a, g)
        e = total_energy(model, state, x, pairs)
        return {"k_x": x, "k_z": state.z.copy(), "k_rot": np.asarray(rot).copy(), "k_g_asm": g_asm,
                "k_a": a, "k_g": g, "k_delta": delta, "k_alpha": alpha, "k_acts": np.array([acts]),
                "k_energy": np.array([e])}
    g_asm = solver._assembled_field(x, state, pairs)
    from tetsolve.local_solver import reduced_collect
    q = reduced_collect(model, solver.factor, rot, g_asm)
    corr = solver._sampled_corrections(x, state, verts, rot)
    a, g = solver._reduced_systems(x, state, verts, g_asm, pairs, rot)
    delta = solver._solve_batch(a, -g)
    alpha, acts = solver._line_search(x, state, verts, delta, pairs, rot, a, g)
    e = total_energy(model, state, x, pairs)
    return {
        "k_x": x, "k_z": state.z.copy(), "k_rot": np.asarray(rot).copy(),
        "k_g_asm": g_asm, "k_q": q, "k_corr": corr, "k_a": a, "k_g": g,
        "k_delta": delta, "k_alpha": alpha, "k_acts": np.array([acts]),
        "k_energy": np.array([e]),
    }


def scene_from_toml(name, frames=None):
    scene = parse_scene(REF / "scenes" / f"{name}.toml")
    model = harness.build_model(scene)
    return scene, model, (frames or scene.frames)


def c1_scene():
    """C1 cantilever: box_grid((24,10,7),(1.2,0.5,0.35)),
    clamp x=0, E=1e6, nu=0.4, rho=1000, h=1/120, s=6, seed 0."""
    mesh = box_grid((24, 10, 7), (1.2, 0.5, 0.35))
    mat = MaterialParams.from_young_poisson(1e6, 0.4, 1000.0)
    fixed = np.flatnonzero(mesh.rest_positions[:, 0] < 1e-9)
    model = Model([(mesh, mat, fixed, np.zeros(3), np.eye(3))])
    scene = parse_scene(REF / "scenes" / "beam.toml")
    scene.h = 1.0 / 120.0
    scene.cubature = CubatureConfig(max_size=6, training_poses=2)
    scene.name = "c1"
    return scene, model


# (frame, sweep) of the per-kernel snapshot: a deformed state, in contact
# for the contact scenes.
SNAPSHOT = {"cube_drop": (20, 2), "two_body": (25, 2), "cube_drop_gs": (20, 2), "two_body_gs": (25, 2),
            "cube_drop_plain": (20, 2), "two_body_plain": (25, 2)}


def gauss_seidel(make):
    """The same scene with scene.solver.mode = "gauss_seidel" (colour sweeps,
    local_solver.py:627-649); the precompute stays per-vertex (harness.py:66-69)."""
    def build():
        scene, model, frames = make()
        scene.solver.mode = "gauss_seidel"
        return scene, model, frames
    return build

def plain(make):
    """The same scene with the plain vertex block descent baseline
    (subspace="none", solver tag plain_local, harness.py:112-113): own-stencil
    systems, no precompute (local_solver.py:325-353, 472-522)."""
    def build():
        scene, model, frames = make()
        scene.solver.subspace = "none"
        return scene, model, frames
    return build


SCENES = {
    "beam": lambda: scene_from_toml("beam"),
    "beam_stiff": lambda: scene_from_toml("beam_stiff", frames=3),
    "cube_drop": lambda: scene_from_toml("cube_drop"),
    "two_body": lambda: scene_from_toml("two_body"),
    "c1": lambda: (*c1_scene(), 3),
    "beam_gs": gauss_seidel(lambda: scene_from_toml("beam", frames=3)),
    "cube_drop_gs": gauss_seidel(lambda: scene_from_toml("cube_drop", frames=24)),
    "two_body_gs": gauss_seidel(lambda: scene_from_toml("two_body", frames=28)),
    "beam_plain": plain(lambda: scene_from_toml("beam", frames=4)),
    "cube_drop_plain": plain(lambda: scene_from_toml("cube_drop", frames=24)),
    "two_body_plain": plain(lambda: scene_from_toml("two_body", frames=28)),
}


def main(names):
    for name in names:
        t0 = time.time()
        scene, model, frames = SCENES[name]()
        is_plain = scene.solver.subspace == "none"
        runtime = (harness.RuntimeData({}, {}, None, None, {}) if is_plain
                   else harness.prepare(model, scene, use_cache=False, seed=scene.seed))
        t_pre = time.time() - t0
        solver = harness.make_solver(model, scene, "plain_local" if is_plain else "jgs2_cubature", runtime)
        cfg = solver.config
        data = {}
        data.update(model_arrays(model))
        if not is_plain:
            data.update(precompute_arrays(runtime.bases, runtime.cubature_sets))
        data["scene_h"] = np.array([scene.h])
        data["scene_cfg"] = np.array([cfg.tol_dx, cfg.max_outer, cfg.max_halvings,
                                      cfg.alpha_floor, float(cfg.local_line_search),
                                      float(cfg.track_energy)])
        t1 = time.time()
        data.update(run_trajectory(model, solver, scene.h, frames,
                                   record_kernels_at=SNAPSHOT.get(name, (2, 1))))
        t_run = time.time() - t1
        data["meta_versions"] = np.array([np.__version__, scipy.__version__])
        data["meta_times"] = np.array([t_pre, t_run])
        np.savez_compressed(OUT / f"{name}.npz", **data)
        iters = data["frame_iterations"]
        print(f"{name}: nv={model.num_vertices} ne={model.num_elements} "
              f"precompute {t_pre:.1f}s run {t_run:.1f}s sweeps {iters.tolist()} "
              f"pairs {data['pairs'].shape[0]}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or list(SCENES))
