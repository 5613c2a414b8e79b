"""GPU parity: the CUDA path (through the C ABI) against the reference's
golden outputs and the CPU oracle on the same inputs.

Tolerances (north_star): positions within 1e-9 relative, identical
iteration counts, bit-exact contact-pair sets; per-kernel intermediates
within the stated relative tolerances below."""

import numpy as np
import pytest

from oracle import jgs2_oracle as orc
from paper_2506_06494_b200.local_solver import LocalSolver, SolverConfig
from helpers import SCENES_SMALL, pair_key, rel_err, replay, scene_inputs

pytestmark = pytest.mark.gpu
ALL = SCENES_SMALL + ("c1",)


def config_of(g, mode="jacobi"):
    c = g["scene_cfg"]
    return SolverConfig(tol_dx=float(c[0]), max_outer=int(c[1]), max_halvings=int(c[2]),
                        alpha_floor=float(c[3]), local_line_search=bool(c[4]),
                        track_energy=bool(c[5]), mode=mode)


def gpu_solver(g, matrix=True, mode="jacobi"):
    model, pre, h = scene_inputs(g)
    if matrix:   # the same Hbar the reference factored (subspace.rest_hessian)
        return model, LocalSolver(model, config_of(g, mode), precompute=pre,
                                  hbar=orc.rest_hessian(model, h)), h
    return model, LocalSolver(model, config_of(g, mode), precompute=pre, h_ref=h), h


@pytest.mark.parametrize("name", ALL)
def test_kernels_match_reference(golden, name):
    g = golden(name)
    model, s, h = gpu_solver(g)
    x, z, rot = g["k_x"], g["k_z"], g["k_rot"]
    assert rel_err(s.rotations(x), rot) < 1e-12
    assert rel_err(s.assembled_field(x, z, h), g["k_g_asm"]) < 1e-12
    assert rel_err(s.collect(rot, g["k_g_asm"]), g["k_q"]) < 1e-11
    corr = s.corrections(x, z, h, rot)
    assert np.abs(corr - g["k_corr"]).max() < 1e-10 * np.abs(g["k_a"]).max()
    a, gg = s.reduced_systems(x, z, h, rot)
    assert rel_err(a, g["k_a"]) < 1e-10
    assert rel_err(gg, g["k_g"]) < 1e-10
    e = s.total_energy(x)
    assert abs(e - g["k_energy"][0]) <= 1e-12 * abs(g["k_energy"][0]) + 1e-300
    assert pair_key(s.find_pairs(x)) == pair_key(orc.find_pairs(model, x).as_rows())


@pytest.mark.parametrize("name", ALL)
def test_trajectory_matches_reference(golden, name):
    g = golden(name)
    model, s, h = gpu_solver(g)

    def sweep(state):
        return s.sweep(state, s.rotations(state.x))

    rep = replay(g, sweep, s.find_pairs)
    assert rep["pair_mismatch"] == 0, rep
    assert rep["iters"] == rep["iters_ref"], rep
    assert rep["pos"] < 1e-9, rep


@pytest.mark.parametrize("name", ("beam", "c1", "two_body"))
def test_outer_solve_matches_reference(golden, name):
    from paper_2506_06494_b200.model import SystemState
    g = golden(name)
    model, s, h = gpu_solver(g)
    for f in range(g["frame_iterations"].size):
        st = SystemState(x=g["frame_x_init"][f].copy(), x_prev=g["frame_x_prev"][f].copy(),
                         v=g["frame_v"][f].copy(), z=g["frame_z"][f].copy(), h=h)
        stats = s.outer_solve(st)
        assert stats.outer_iterations == int(g["frame_iterations"][f])
        assert stats.converged == bool(g["frame_converged"][f])
        assert rel_err(st.x, g["frame_x_final"][f]) < 1e-9


@pytest.mark.parametrize("name", ("beam", "c1"))
def test_device_assembled_factor_matches_reference_collect(golden, name):
    g = golden(name)
    _, s, _ = gpu_solver(g, matrix=False)
    assert rel_err(s.collect(g["k_rot"], g["k_g_asm"]), g["k_q"]) < 1e-11
    assert s.factor_info.nnz_dof > 0


def test_bit_identical_reruns(golden):
    g = golden("two_body")
    outs = []
    for _ in range(2):
        model, s, h = gpu_solver(g)
        from paper_2506_06494_b200.model import SystemState
        xs = []
        for f in range(0, 30, 3):
            st = SystemState(x=g["frame_x_init"][f].copy(), x_prev=g["frame_x_prev"][f].copy(),
                             v=g["frame_v"][f].copy(), z=g["frame_z"][f].copy(), h=h)
            s.outer_solve(st)
            xs.append(st.x)
        outs.append(np.stack(xs))
        s.close()
    assert np.array_equal(outs[0], outs[1])


# ------------------------------------------------ multi-body contact at scale
def _c4_small(cells, touching=True):
    # the tank packed so neighbouring balls touch (c4t): cross-body
    # vertex-triangle pairs active from the first sweep
    from paper_2506_06494_b200 import scenes
    from paper_2506_06494_b200.precompute import Precompute
    m, st, h, _ = scenes.build(f"c4{'t' if touching else 's'}{cells}")
    return m, st, h, Precompute.injected(m, h)


def test_grid_broadphase_pairs_match_bruteforce():
    """Spatial-grid candidates + reference-rounding narrowphase give the
    brute-force pair set exactly (contact.py:216-240), on 10 bodies."""
    m, st, h, pre = _c4_small(10)
    s = LocalSolver(m, SolverConfig(), precompute=pre, h_ref=h)
    rng = np.random.default_rng(3)
    for k in range(3):
        x = st.x + (0 if k == 0 else 2e-3 * rng.standard_normal(st.x.shape))
        got = s.find_pairs(x)
        ref = orc.find_pairs(m, x).as_rows()
        assert len(ref) > 0
        assert pair_key(got) == pair_key(ref)
        assert np.array_equal(got[:, 6], ref[:, 6])  # distances bit-identical


def test_contact_sweeps_match_oracle():
    """Two JGS2 sweeps with plane + vertex-triangle contact on 10 bodies:
    GPU vs CPU oracle (same injected precompute, same Hbar). The oracle's
    brute-force find_pairs runs once per backtracking trial, so each oracle
    sweep costs minutes on the GPU box's host."""
    from paper_2506_06494_b200.model import SystemState
    m, st, h, pre = _c4_small(6)
    hbar = orc.rest_hessian(m, h)
    s = LocalSolver(m, SolverConfig(), precompute=pre, hbar=hbar)
    o = orc.OracleSolver(m, pre, h, orc.OracleConfig(), factor=orc.rest_factor(hbar))
    a = SystemState(x=st.x.copy(), x_prev=st.x_prev.copy(), v=st.v.copy(), z=st.z.copy(), h=h)
    b = SystemState(x=st.x.copy(), x_prev=st.x_prev.copy(), v=st.v.copy(), z=st.z.copy(), h=h)
    for _ in range(2):
        assert pair_key(s.find_pairs(a.x)) == pair_key(orc.find_pairs(m, b.x).as_rows())
        dxa, ia = s.sweep(a, s.rotations(a.x))
        dxb, ib = o.sweep(b, orc.vertex_rotations(m, b.x))
        assert ia["line_search_activations"] == ib["line_search_activations"]
        assert rel_err(a.x, b.x) < 1e-9


@pytest.mark.parametrize("name", ("beam", "two_body", "cube_drop"))
def test_device_frame_driver_matches_reference(golden, name):
    """compute_z + capped initialize_step + outer_solve + velocity update
    fully on the device (harness.py:187-202) reproduce the reference
    trajectory frame by frame."""
    from paper_2506_06494_b200.model import SystemState
    g = golden(name)
    model, s, h = gpu_solver(g)
    st = SystemState.initial(model, h)
    s.set_frame_state(st, model.gravity)
    for f in range(g["frame_iterations"].size):
        (it, conv), = s.run_frames(1)
        assert it == int(g["frame_iterations"][f]), (f, it)
        assert rel_err(s.get_x(), g["frame_x_final"][f]) < 1e-9


@pytest.mark.parametrize("name", ("beam", "two_body", "cube_drop"))
def test_host_timestep_matches_reference(golden, name):
    """One ABI call per frame from host buffers (jgs2_timestep_host): the
    reference trajectory frame by frame, iteration counts identical, and the
    velocity update v = (x - x_prev) / h."""
    from paper_2506_06494_b200.model import SystemState
    g = golden(name)
    model, s, h = gpu_solver(g)
    st = SystemState.initial(model, h)
    for f in range(g["frame_iterations"].size):
        xp = st.x_prev.copy()
        it, conv = s.timestep(st, model.gravity)
        assert it == int(g["frame_iterations"][f]), (f, it)
        assert rel_err(st.x_prev, g["frame_x_final"][f]) < 1e-9
        np.testing.assert_array_equal(st.v, (st.x_prev - xp) / h)


@pytest.mark.parametrize("name", ("beam_gs", "cube_drop_gs", "two_body_gs"))
def test_gauss_seidel_trajectory_matches_reference(golden, name):
    # colour sweeps (local_solver.py:627-649) against the reference's own
    # gauss_seidel trajectories: per-colour pair re-detection and local
    # search, sweep-start collect and corrections
    g = golden(name)
    model, s, h = gpu_solver(g, mode="gauss_seidel")

    def sweep(state):
        return s.sweep(state, s.rotations(state.x))

    rep = replay(g, sweep, s.find_pairs)
    assert rep["pair_mismatch"] == 0, rep
    assert rep["iters"] == rep["iters_ref"], rep
    assert rep["pos"] < 1e-9, rep


def _gs_pair(name):
    from paper_2506_06494_b200 import scenes
    from paper_2506_06494_b200.model import SystemState
    from paper_2506_06494_b200.precompute import Precompute
    m, st, h, _ = scenes.build(name)
    pre = Precompute.injected(m, h, samples=6, seed=0)
    cfg = SolverConfig(tol_dx=m.tol_dx, mode="gauss_seidel")
    s = LocalSolver(m, cfg, precompute=pre, hbar=orc.rest_hessian(m, h))
    o = orc.OracleSolver(m, pre, h, orc.OracleConfig(tol_dx=m.tol_dx, mode="gauss_seidel"))
    cp = lambda: SystemState(x=st.x.copy(), x_prev=st.x_prev.copy(), v=st.v.copy(),  # noqa: E731
                             z=st.z.copy(), h=h)
    return m, s, o, cp(), cp()


def test_gauss_seidel_contact_sweeps_match_oracle():
    # ten-body tank (C4 construction at 6 cells/ball, floor + wall pairs):
    # GS colour sweeps against the oracle's GS on the same inputs
    m, s, o, sg, so = _gs_pair("c4s6")
    for _ in range(2):
        rot = orc.vertex_rotations(m, so.x)
        dxo, io = o.sweep(so, rot)
        dxg, ig = s.sweep(sg, s.rotations(sg.x))
        assert rel_err(sg.x, so.x) < 1e-9
        assert ig["line_search_activations"] == io["line_search_activations"]


def test_gauss_seidel_penetration_raises_like_reference():
    # touching tank: the per-colour updates carry no feasibility cap
    # (local_solver.py:641-647), so a colour can push a vertex through a
    # triangle; the reference's barrier then raises FeasibilityError
    # (energy.py:205-221) -- the GPU path raises it in the same sweep
    from paper_2506_06494_b200.local_solver import FeasibilityError
    m, s, o, sg, so = _gs_pair("c4t6")
    for k in range(3):
        try:
            o.sweep(so, orc.vertex_rotations(m, so.x))
            ref_raised = False
        except orc.Infeasible:
            ref_raised = True
        if ref_raised:
            with pytest.raises(FeasibilityError):
                s.sweep(sg, s.rotations(sg.x))
            return
        s.sweep(sg, s.rotations(sg.x))
        assert rel_err(sg.x, so.x) < 1e-9
    pytest.skip("no penetration within 3 sweeps")


def test_nonfinite_state_rejected_and_solver_unharmed():
    # NaN positions raise ValueError on the host (on the device they would
    # poison the context); the solver's next sweep equals a fresh solver's
    from paper_2506_06494_b200 import scenes
    from paper_2506_06494_b200.model import SystemState
    from paper_2506_06494_b200.precompute import Precompute
    m, st, h, _ = scenes.build("c4s6")
    pre = Precompute.injected(m, h, samples=6, seed=0)
    cp = lambda: SystemState(x=st.x.copy(), x_prev=st.x_prev.copy(), v=st.v.copy(),  # noqa: E731
                             z=st.z.copy(), h=h)
    cfg = SolverConfig(tol_dx=m.tol_dx)
    s = LocalSolver(m, cfg, precompute=pre, h_ref=h)
    bad = cp()
    bad.x[5] = np.nan
    with pytest.raises(ValueError):
        s.sweep(bad)
    with pytest.raises(ValueError):
        s.outer_solve(bad)
    s2 = LocalSolver(m, cfg, precompute=pre, h_ref=h)
    a, b = cp(), cp()
    dxa, _ = s.sweep(a, s.rotations(a.x))
    dxb, _ = s2.sweep(b, s2.rotations(b.x))
    assert np.array_equal(a.x, b.x)
    assert np.array_equal(dxa, dxb)


def test_run_frames_from_reference_cache_matches_reference(golden, tmp_path):
    # harness.run-style frames on the GPU solver, precompute loaded from the
    # cache files the reference wrote; outputs in the reference's formats
    from pathlib import Path
    from paper_2506_06494_b200 import formats
    from paper_2506_06494_b200.model import Model, SystemState
    io = Path(__file__).resolve().parent / "golden" / "io"
    g = golden("beam")
    model = Model.from_arrays(g)
    pre, info = formats.load_precompute_cache(io / "beam_bases.npz", io / "beam_cubature.npz")
    h = float(g["scene_h"][0])
    s = LocalSolver(model, config_of(g), precompute=pre, hbar=orc.rest_hessian(model, h))
    state = SystemState.initial(model, h)
    nf = int(g["frame_iterations"].size)
    failed = formats.run_frames(model, s, state, nf, tmp_path)
    assert failed == []
    assert rel_err(state.x_prev, g["frame_x_final"][nf - 1]) < 1e-9
    rows = formats.read_metrics(tmp_path / "metrics.csv")
    assert len(rows) == int(g["frame_iterations"].sum())
    assert (tmp_path / f"frame_{nf:04d}.obj").exists() and (tmp_path / f"body0_frame_{nf:04d}.node").exists()


@pytest.mark.parametrize("name", ("beam", "c1", "two_body"))
def test_drop_in_reference_objects_match_reference(golden, name):
    """The reference's own call (harness.make_solver, harness.py:120-127):
    LocalSolver(model, config, bases={v: PerturbationBasis},
    cubature_sets={v: CubatureSet}, factor=<SciPy SuperLU of Hbar>). The
    matrix is recovered from the factor on the mesh pattern
    (hbar_from_factor) and re-factored on the device; every golden frame
    from its frame-start state reproduces the reference."""
    import scipy.sparse.linalg as spla
    from helpers import reference_objects
    from paper_2506_06494_b200.model import SystemState
    g = golden(name)
    model, pre, h = scene_inputs(g)
    bases, sets = reference_objects(pre)
    lu = spla.splu(orc.rest_hessian(model, h).tocsc())
    s = LocalSolver(model, config_of(g), bases, sets, lu)
    for f in range(g["frame_iterations"].size):
        st = SystemState(x=g["frame_x_init"][f].copy(), x_prev=g["frame_x_prev"][f].copy(),
                         v=g["frame_v"][f].copy(), z=g["frame_z"][f].copy(), h=h)
        stats = s.outer_solve(st)
        assert stats.outer_iterations == int(g["frame_iterations"][f])
        assert rel_err(st.x, g["frame_x_final"][f]) < 1e-9


@pytest.mark.parametrize("name", ("beam_plain", "cube_drop_plain", "two_body_plain"))
def test_plain_vbd_trajectory_matches_reference(golden, name):
    """subspace="none" (the reference's plain vertex block descent baseline,
    local_solver.py:325-353, 472-522) against the reference's own plain_local
    trajectories: pair sets, sweeps per frame, positions."""
    from paper_2506_06494_b200.model import Model
    g = golden(name)
    model = Model.from_arrays(g)
    h = float(g["scene_h"][0])
    c = g["scene_cfg"]
    cfg = SolverConfig(tol_dx=float(c[0]), max_outer=int(c[1]), max_halvings=int(c[2]),
                       alpha_floor=float(c[3]), local_line_search=bool(c[4]), track_energy=bool(c[5]),
                       subspace="none")
    s = LocalSolver(model, cfg)

    def sweep(state):
        return s.sweep(state)

    rep = replay(g, sweep, s.find_pairs)
    assert rep["pair_mismatch"] == 0, rep
    assert rep["iters"] == rep["iters_ref"], rep
    assert rep["pos"] < 1e-9, rep


@pytest.mark.parametrize("name", ("cube_drop_plain", "two_body_plain"))
def test_plain_vbd_kernels_match_reference(golden, name):
    from paper_2506_06494_b200.model import Model
    g = golden(name)
    model = Model.from_arrays(g)
    h = float(g["scene_h"][0])
    s = LocalSolver(model, SolverConfig(subspace="none"))
    x, z = g["k_x"], g["k_z"]
    a, gg = s.reduced_systems(x, z, h, g["k_rot"])
    assert rel_err(a, g["k_a"]) < 1e-10
    assert rel_err(gg, g["k_g"]) < 1e-10
    d, al, acts = s.local_step(x, z, h, g["k_rot"])
    assert rel_err(d, g["k_delta"]) < 1e-10
    np.testing.assert_allclose(al, g["k_alpha"], rtol=1e-12)
    assert acts == int(g["k_acts"][0])
