"""Scalable precompute on the device (precompute_gpu.py)
against the reference's own C1 precompute (tests/golden/c1.npz: bases
written by tetsolve.subspace.precompute_bases + retain_rows) and a dense
inverse of the rest Hessian."""

import ctypes as C

import numpy as np
import pytest

from oracle import jgs2_oracle as orc
from helpers import scene_inputs

pytestmark = pytest.mark.gpu


def _ctx_with_selinv(model, h):
    from paper_2506_06494_b200 import _lib as L
    from paper_2506_06494_b200.local_solver import upload_model
    lib = L.lib()
    ctx = lib.jgs2_create(0)
    keep = []
    upload_model(lib, ctx, model, keep)
    fi = L.FactorInfo()
    L.check(lib.jgs2_factor_rest(ctx, h, 32, C.byref(fi)), ctx)  # METIS ordering (default)
    L.check(lib.jgs2_selected_inverse(ctx, None), ctx)
    return lib, ctx


@pytest.mark.parametrize("name", ("beam", "two_body"))
def test_selected_inverse_matches_dense_inverse(golden, name):
    # every block on the filled pattern equals the dense (Hbar^-1)_{wv}
    from paper_2506_06494_b200.precompute_gpu import inverse_blocks
    g = golden(name)
    model, _, h = scene_inputs(g)
    hb = orc.rest_hessian(model, h).toarray()
    zi = np.linalg.inv(hb)
    lib, ctx = _ctx_with_selinv(model, h)
    try:
        nv = model.num_vertices
        vv, ww = np.meshgrid(np.arange(nv), np.arange(nv), indexing="ij")
        out, found = inverse_blocks(lib, ctx, vv.ravel(), ww.ravel())
        # ref[v * nv + w] = zi[3w:3w+3, 3v:3v+3] (rows of w, columns of v)
        ref = zi.reshape(nv, 3, nv, 3).transpose(2, 0, 1, 3).reshape(nv * nv, 3, 3)
        assert found.mean() > 0.2  # the pattern (fill included) covers a good part of a small mesh
        fixed = np.asarray(model.fixed_mask)
        sel = found & ~(fixed[vv.ravel()] & fixed[ww.ravel()])  # fixed-fixed: identity rows of Hbar
        err = np.abs(out[sel] - ref[sel]).max() / np.abs(zi).max()
        assert err < 1e-12, err
        adj = (np.abs(hb.reshape(nv, 3, nv, 3)).sum(axis=(1, 3)) > 0)
        free_pairs = ~fixed[vv.ravel()] & ~fixed[ww.ravel()]
        assert np.all(found[adj.ravel() & free_pairs])  # every mesh neighbour is on the pattern
    finally:
        lib.jgs2_destroy(ctx)


def test_bases_match_reference_c1(golden):
    """Gbar_v, gbar_rows and the retained rows of the own vertex and its
    incident elements equal the reference's C1 bases (subspace.py:133-203)."""
    from paper_2506_06494_b200.precompute_gpu import scalable_precompute
    g = golden("c1")
    model, ref, h = scene_inputs(g)
    pre, info = scalable_precompute(model, h, max_size=6, training_poses=2)
    np.testing.assert_array_equal(pre.vertices, ref.vertices)
    scale = np.abs(ref.gbar).max()
    assert np.abs(pre.gbar - ref.gbar).max() < 1e-12 * scale
    assert np.abs(pre.gbar_rows - ref.gbar_rows[:, :, :3]).max() < 1e-12 * scale
    tets = np.asarray(model.tets)
    inc = [set() for _ in range(model.num_vertices)]
    for e, t in enumerate(tets):
        for w in t:
            inc[w].update(int(u) for u in t)
    checked = 0
    for k in range(ref.vertices.size):
        v = int(ref.vertices[k])
        rk = dict(zip(ref.vrows_keys[ref.vrows_ptr[k]:ref.vrows_ptr[k + 1]].tolist(),
                      ref.vrows[ref.vrows_ptr[k]:ref.vrows_ptr[k + 1]]))
        pk = dict(zip(pre.vrows_keys[pre.vrows_ptr[k]:pre.vrows_ptr[k + 1]].tolist(),
                      pre.vrows[pre.vrows_ptr[k]:pre.vrows_ptr[k + 1]]))
        for w in inc[v] | {v}:
            assert np.abs(pk[w] - rk[w]).max() < 1e-12 * max(np.abs(rk[w]).max(), 1.0), (v, w)
            checked += 1
    assert checked > 10 * ref.vertices.size
    # cubature sets: nonnegative weights, corners retained, mostly at the target
    assert np.all(pre.cub_weights > 0)
    # the candidate pool is the vertex's front (train.cuh): most, not all, reach the target
    assert info["converged_fraction"] >= 0.85, info["converged_fraction"]


def test_scalable_precompute_runs_the_reference_c1_frames(golden):
    """The device precompute drives the C1 cantilever like the reference's own
    precompute: every frame converges, in a comparable number of sweeps."""
    from paper_2506_06494_b200.local_solver import LocalSolver, SolverConfig
    from paper_2506_06494_b200.model import SystemState
    from paper_2506_06494_b200.precompute_gpu import scalable_precompute
    g = golden("c1")
    model, _, h = scene_inputs(g)
    pre, _ = scalable_precompute(model, h)
    s = LocalSolver(model, SolverConfig(), precompute=pre, h_ref=h)
    for f in range(g["frame_iterations"].size):
        st = SystemState(x=g["frame_x_init"][f].copy(), x_prev=g["frame_x_prev"][f].copy(),
                         v=g["frame_v"][f].copy(), z=g["frame_z"][f].copy(), h=h)
        stats = s.outer_solve(st)
        assert stats.converged
        assert stats.outer_iterations <= 3 * int(g["frame_iterations"][f]) + 2
