"""GPU parity at scale: the CUDA path against the CPU oracle's fixtures
(tests/golden/make_scale_goldens.py) on scaled-down BASELINE constructions
-- the C4 tank at 12 cells/ball (plane + wall contact), the touching C4 tank
at 8 cells/ball (cross-body vertex-triangle pairs), C3 at half resolution
(125K tets, no contact) and C2 at 20 cells.

Each frame starts from the oracle's previous frame (harness.py:187-211:
compute_z, the feasibility-capped predictor, outer_solve to tol_dx). Bar
(north_star): positions within 1e-9 relative, identical sweeps per frame
and identical backtracking halvings per sweep; the feasibility cap within
1e-12 relative."""

from pathlib import Path

import numpy as np
import pytest

from oracle import jgs2_oracle as orc
from paper_2506_06494_b200 import scenes
from paper_2506_06494_b200.local_solver import LocalSolver, SolverConfig
from paper_2506_06494_b200.model import SystemState
from paper_2506_06494_b200.precompute import Precompute
from helpers import rel_err

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden"


def load(name):
    p = GOLDEN / f"scale_{name}.npz"
    if not p.exists():
        pytest.skip(f"{p.name} not generated")
    with np.load(p) as d:
        return {k: d[k] for k in d.files}


@pytest.mark.parametrize("name", ("c4s12", "c4t8", "c3s2", "c2s20"))
def test_scale_frames_match_oracle(name):
    g = load(name)
    m, _, h, _ = scenes.build(name)
    assert m.num_vertices == int(g["nv"][0]) and m.num_elements == int(g["ne"][0])
    pre = Precompute.injected(m, h, samples=6, seed=0)
    tol = float(g["tol_dx"][0])
    s = LocalSolver(m, SolverConfig(tol_dx=tol, max_outer=500), precompute=pre,
                    hbar=orc.rest_hessian(m, h))
    xf = g["frame_x_final"]
    sweep_frame = g["sweep_frame"]
    x_prev = np.array(m.initial_positions, dtype=np.float64)
    v = np.zeros_like(x_prev)
    productive = False
    for f in range(xf.shape[0]):
        z = orc.compute_z(m, x_prev, v, h)
        dz = z - x_prev
        cap = s.step_cap(x_prev, dz)
        assert abs(cap - g["frame_cap"][f]) <= 1e-12 * max(abs(g["frame_cap"][f]), 1e-300), (f, cap)
        st = SystemState(x=x_prev + g["frame_cap"][f] * dz, x_prev=x_prev, v=v, z=z, h=h)
        if f == 0:  # per-sweep positions of the first two sweeps
            st1 = SystemState(x=st.x.copy(), x_prev=x_prev, v=v, z=z, h=h)
            for k in range(min(2, len(g["sweep_x"]))):
                s.sweep(st1, s.rotations(st1.x))
                assert rel_err(st1.x, g["sweep_x"][k]) < 1e-9, (k,)
        stats = s.outer_solve(st)
        sel = sweep_frame == f
        assert stats.outer_iterations == int(g["frame_iterations"][f]), (f, stats.outer_iterations)
        assert stats.line_search_activations == [int(a) for a in g["sweep_halvings"][sel]], f
        # energies: E moves by |grad E| |x - x_oracle| ~ 1e-9 relative where the
        # factor solves round differently (device Cholesky vs SuperLU)
        np.testing.assert_allclose(stats.energies, g["sweep_energy"][sel], rtol=1e-8)
        assert rel_err(st.x, xf[f]) < 1e-9, f
        productive |= bool(np.any(g["sweep_halvings"][sel] <= 10))
        v = (xf[f] - x_prev) / h
        x_prev = xf[f].copy()
    assert productive  # at least one accepted sweep with gamma > cap 2^-10


@pytest.mark.parametrize("name,scales", [("c4t8", (1e-4, 1e-2, 1.0, 100.0)), ("c4s12", (1e-3, 1.0))])
def test_step_cap_matches_oracle(name, scales):
    """feasibility_step_cap (assembly.py:263-291) on the device -- planes, the
    pair-table bound and the hierarchical-grid radius rounds -- against the
    oracle for small to body-sized random steps."""
    m, st, h, _ = scenes.build(name)
    pre = Precompute.injected(m, h, samples=6, seed=0)
    s = LocalSolver(m, SolverConfig(), precompute=pre, h_ref=h)
    ext = float(np.ptp(m.initial_positions, axis=0).max())
    rng = np.random.default_rng(7)
    orc.PRUNE = True
    try:
        for sc in scales:
            for trial in range(2):
                dx = sc * ext * rng.standard_normal(st.x.shape)
                if trial == 1:  # moving surfaces only toward the neighbour balls
                    dx[:, 1] = np.abs(dx[:, 1])
                a = s.step_cap(st.x, dx)
                b = orc.feasibility_cap(m, st.x, dx)
                assert abs(a - b) <= 1e-12 * b, (sc, trial, a, b)
    finally:
        orc.PRUNE = False


@pytest.mark.parametrize("name", ("two_body", "cube_drop", "c1"))
def test_local_steps_match_reference(golden, name):
    """delta (batched gesv), alpha (local search) and activations against the
    reference's own k_delta / k_alpha / k_acts snapshots."""
    from helpers import scene_inputs
    g = golden(name)
    model, pre, h = scene_inputs(g)
    s = LocalSolver(model, SolverConfig(), precompute=pre, hbar=orc.rest_hessian(model, h))
    d, al, acts = s.local_step(g["k_x"], g["k_z"], h, g["k_rot"])
    assert rel_err(d, g["k_delta"]) < 1e-10
    np.testing.assert_array_equal(al, g["k_alpha"])
    assert acts == int(g["k_acts"][0])


def test_local_steps_match_oracle_with_contact():
    """The same at a contact state of the touching tank, where the alpha caps
    bind (plane and vertex-triangle rates, local_solver.py:450-470)."""
    m, st, h, _ = scenes.build("c4t6")
    pre = Precompute.injected(m, h, samples=6, seed=0)
    hbar = orc.rest_hessian(m, h)
    s = LocalSolver(m, SolverConfig(), precompute=pre, hbar=hbar)
    o = orc.OracleSolver(m, pre, h, factor=orc.rest_factor(hbar))
    rot = orc.vertex_rotations(m, st.x)
    d, al, acts = s.local_step(st.x, st.z, h, rot)
    pairs = orc.find_pairs(m, st.x)
    verts = o.p.free
    ga = o.assembled_field(st.x, st.z, h, pairs)
    a, gg = o.reduced_systems(st.x, st.z, h, verts, ga, pairs, rot)
    delta = o.solve3(a, -gg)
    alpha, acts_o = o.line_search(st.x, verts, delta, pairs, a, gg)
    assert rel_err(d, delta) < 1e-9
    # alpha = 0.9 d / (2 |delta|) inherits delta's 1e-9 relative agreement
    np.testing.assert_allclose(al, alpha, rtol=1e-9)
    assert np.any(alpha < 1.0)
    assert acts == acts_o
