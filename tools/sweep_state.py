"""Run K device-resident sweeps of a scene and save x (bitwise A/B of env-selected schedules).

usage: python tools/sweep_state.py <scene> <sweeps> <out.npy>   (env selects the schedule)"""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit('/', 2)[0])
from paper_2506_06494_b200 import scenes  # noqa: E402
from paper_2506_06494_b200.local_solver import LocalSolver, SolverConfig  # noqa: E402
from paper_2506_06494_b200.model import SystemState  # noqa: E402
from paper_2506_06494_b200.precompute import Precompute  # noqa: E402

name, k, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
m, st, h, _ = scenes.build(name)
pre = Precompute.injected(m, h, samples=6, seed=0)
s = LocalSolver(m, SolverConfig(max_outer=500, tol_dx=getattr(m, "tol_dx", 1e-3)), precompute=pre, h_ref=h)
init = SystemState(x=st.x_prev.copy(), x_prev=st.x_prev.copy(), v=st.v.copy(), z=st.z.copy(), h=h)
s.set_frame_state(init, m.gravity)
s.run_sweeps(k)
x = s.get_x()
np.save(out, x)
print(name, k, "sweeps, |x| =", float(np.abs(x).sum()))
