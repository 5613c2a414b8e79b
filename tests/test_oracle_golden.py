"""Pin the CPU oracle against the reference's own outputs (golden fixtures).

CPU only. These tests are what make the oracle trustworthy as the checker of
the CUDA path."""

import numpy as np
import pytest

from oracle import jgs2_oracle as orc
from paper_2506_06494_b200.model import box_grid
from helpers import SCENES_SMALL, replay, rel_err, scene_inputs


def make_solver(g):
    model, pre, h = scene_inputs(g)
    cfg = g["scene_cfg"]
    oc = orc.OracleConfig(tol_dx=float(cfg[0]), max_outer=int(cfg[1]),
                          max_halvings=int(cfg[2]), alpha_floor=float(cfg[3]))
    return model, orc.OracleSolver(model, pre, h, oc), h


@pytest.mark.parametrize("name,div,ext", [("beam", (8, 3, 3), (0.4, 0.15, 0.15)),
                                          ("c1", (24, 10, 7), (1.2, 0.5, 0.35))])
def test_box_grid_matches_reference_mesh(golden, name, div, ext):
    g = golden(name)
    mesh = box_grid(div, ext)
    assert np.array_equal(mesh.tets, g["model_tets"])
    assert rel_err(mesh.rest_positions, g["model_rest_positions"]) < 1e-15
    assert rel_err(mesh.dm_inv, g["model_dm_inv"]) < 1e-13
    assert rel_err(mesh.rest_volumes, g["model_volumes"]) < 1e-13
    assert np.array_equal(mesh.surface_tris, g["model_surface_tris"])


@pytest.mark.parametrize("name", SCENES_SMALL + ("c1",))
def test_oracle_kernels_match_reference(golden, name):
    g = golden(name)
    model, solver, h = make_solver(g)
    x, z = g["k_x"], g["k_z"]
    rot = orc.vertex_rotations(model, x)
    assert rel_err(rot, g["k_rot"]) < 1e-12
    pairs = orc.find_pairs(model, x)
    g_asm = solver.assembled_field(x, z, h, pairs)
    assert rel_err(g_asm, g["k_g_asm"]) < 1e-12
    q = solver.collect(g["k_rot"], g["k_g_asm"])
    assert rel_err(q, g["k_q"]) < 1e-12
    corr = solver.corrections(x, solver.p.free, g["k_rot"])
    assert rel_err(corr, g["k_corr"]) < 1e-11
    a, gg = solver.reduced_systems(x, z, h, solver.p.free, g["k_g_asm"], pairs, g["k_rot"])
    assert rel_err(a, g["k_a"]) < 1e-11
    assert rel_err(gg, g["k_g"]) < 1e-11
    delta = solver.solve3(g["k_a"], -g["k_g"])
    assert rel_err(delta, g["k_delta"]) < 1e-12
    alpha, acts = solver.line_search(x, solver.p.free, g["k_delta"], pairs, g["k_a"], g["k_g"])
    assert np.array_equal(alpha, g["k_alpha"]) and acts == int(g["k_acts"][0])
    e = orc.total_energy(model, z, h, x, pairs)
    assert abs(e - g["k_energy"][0]) <= 1e-12 * abs(g["k_energy"][0])


@pytest.mark.parametrize("name", SCENES_SMALL + ("c1",))
def test_oracle_trajectory_matches_reference(golden, name):
    g = golden(name)
    model, solver, h = make_solver(g)

    def sweep(state):
        rot = orc.vertex_rotations(model, state.x)
        return solver.sweep(state, rot)

    rep = replay(g, sweep, lambda x: orc.find_pairs(model, x).as_rows())
    assert rep["iters"] == rep["iters_ref"]
    assert rep["pair_mismatch"] == 0
    assert rep["pos"] < 1e-9, rep


def test_barrier_known_answer():
    # test_energy.py:132-136 known value at d=0.5, dhat=kappa=1
    b, _, _ = orc.barrier(0.5, 1.0, 1.0)
    assert b == pytest.approx(0.17328679513998632, rel=1e-15)


GS_SCENES = ("beam_gs", "cube_drop_gs", "two_body_gs")


@pytest.mark.parametrize("name", GS_SCENES)
def test_oracle_gauss_seidel_trajectory_matches_reference(golden, name):
    # scene.solver.mode = "gauss_seidel" goldens (local_solver.py:627-649)
    g = golden(name)
    model, solver, h = make_solver(g)
    solver.cfg.mode = "gauss_seidel"

    def sweep(state):
        rot = orc.vertex_rotations(model, state.x)
        return solver.sweep(state, rot)

    rep = replay(g, sweep, lambda x: orc.find_pairs(model, x).as_rows())
    assert rep["iters"] == rep["iters_ref"]
    assert rep["pair_mismatch"] == 0
    assert rep["pos"] < 1e-9, rep


def test_gauss_seidel_equals_jacobi_without_contact(golden):
    # bitwise equal to Jacobi when there is no contact
    gs, jac = golden("beam_gs"), golden("beam")
    n = gs["traj_x"].shape[0]
    assert np.array_equal(gs["traj_x"], jac["traj_x"][:n])


def test_oracle_pruning_is_exact():
    """The oracle's spatial pruning (used to generate the scale fixtures)
    returns the brute-force pair table and feasibility cap bit for bit."""
    from paper_2506_06494_b200 import scenes
    m, st, h, _ = scenes.build("c4t6")
    rng = np.random.default_rng(5)
    x = st.x + 5e-4 * rng.standard_normal(st.x.shape)
    dx = 0.05 * rng.standard_normal(st.x.shape)
    try:
        orc.PRUNE = False
        a, ca = orc.find_pairs(m, x).as_rows(), orc.feasibility_cap(m, x, dx)
        orc.PRUNE = True
        b, cb = orc.find_pairs(m, x).as_rows(), orc.feasibility_cap(m, x, dx)
    finally:
        orc.PRUNE = False
    assert (a[:, 0] == 1).sum() > 0
    np.testing.assert_array_equal(a, b)
    assert ca == cb
