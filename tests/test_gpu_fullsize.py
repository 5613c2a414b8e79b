"""Full-size GPU checks at BASELINE.json configs[1] (C2: one ~350K-tet puffer
ball dropping onto a ground plane with the IPC barrier).

At this size the CPU oracle cannot run sweeps in test time, so the checks are
size-independent properties plus the parts the oracle can still do exactly:
  * the contact pair set after every sweep equals the oracle's find_pairs
    (contact.py:216-240; one body, so plane pairs over ~60K surface vertices),
    bit-exact rows and distances;
  * every active barrier distance stays > 0 (feasibility, energy.py:205-221);
  * an accepted backtracking trial does not raise the total energy beyond the
    reference's 1e-12 slack (local_solver.py:566-571);
  * whole timesteps from host buffers are bit-identical across two fresh
    contexts (deterministic reductions, no FP atomics).
"""

import numpy as np
import pytest

from oracle import jgs2_oracle as orc
from paper_2506_06494_b200 import scenes
from paper_2506_06494_b200.local_solver import LocalSolver, SolverConfig
from paper_2506_06494_b200.model import SystemState
from paper_2506_06494_b200.precompute import Precompute
from helpers import pair_key

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c2():
    m, st, h, _ = scenes.build("c2")
    return m, st, h, Precompute.injected(m, h, samples=6, seed=0)


def _solver(m, h, pre):
    return LocalSolver(m, SolverConfig(max_outer=500, tol_dx=m.tol_dx), precompute=pre, h_ref=h)


def _frames(s, m, st, h, n):
    fs = SystemState(x=None, x_prev=st.x_prev.copy(), v=st.v.copy(), z=None, h=h)
    iters = []
    for _ in range(n):
        it, _ = s.timestep(fs, m.gravity)
        iters.append(it)
    return fs.x_prev.copy(), fs.v.copy(), iters


def test_c2_timesteps_bit_identical(c2):
    m, st, h, pre = c2
    assert m.num_elements > 300_000
    runs = []
    for _ in range(2):
        s = _solver(m, h, pre)
        runs.append(_frames(s, m, st, h, 2))
        s.close()
    (xa, va, ia), (xb, vb, ib) = runs
    assert ia == ib
    assert np.array_equal(xa, xb) and np.array_equal(va, vb)
    assert np.all(np.isfinite(xa))


def test_c2_sweeps_pairs_exact_feasible_energy_guard(c2):
    m, st, h, pre = c2
    s = _solver(m, h, pre)
    xp, v, _ = _frames(s, m, st, h, 1)       # one frame in: the ball is in contact range
    g = np.asarray(m.gravity, dtype=np.float64)
    z = xp + h * v + (h * h) * g
    state = SystemState(x=xp.copy(), x_prev=xp.copy(), v=v.copy(), z=z, h=h)
    for _ in range(3):
        got = s.find_pairs(state.x)
        ref = orc.find_pairs(m, state.x).as_rows()
        assert pair_key(got) == pair_key(ref)
        assert np.array_equal(got[:, 6], ref[:, 6])          # distances bit-identical
        assert np.all(got[:, 6] > 0.0)
        s.set_state(state.x, state.z, h)
        e0 = s.total_energy(state.x)
        _, info = s.sweep(state, s.rotations(state.x))
        if info["halvings"] <= 30:                            # a trial was accepted
            assert info["energy"] <= e0 + 1e-12 * abs(e0), (info["energy"], e0)
        assert np.all(np.isfinite(state.x))
    got = s.find_pairs(state.x)
    assert np.all(got[:, 6] > 0.0)
    s.close()
