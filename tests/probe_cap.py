"""Diagnostic (not a test): cost and inputs of the feasibility cap on a contact scene."""
import sys
import time
import numpy as np
sys.path.insert(0, ".")
from paper_2506_06494_b200 import scenes
from paper_2506_06494_b200.local_solver import LocalSolver, SolverConfig
from paper_2506_06494_b200.precompute import Precompute
from paper_2506_06494_b200.model import SystemState
name = sys.argv[1] if len(sys.argv) > 1 else "c4"
m, st, h, d = scenes.build(name)
pre = Precompute.injected(m, h)
s = LocalSolver(m, SolverConfig(tol_dx=getattr(m, "tol_dx", 1e-3)), precompute=pre, h_ref=h)
init = SystemState(x=st.x_prev.copy(), x_prev=st.x_prev.copy(), v=st.v.copy(), z=st.z.copy(), h=h)
s.set_frame_state(init, m.gravity)
sv = m.surface_vertices
print("dhat", m.barrier.dhat, "nsv", len(sv), "nst", len(m.surface_tris), flush=True)
for f in range(int(sys.argv[2]) if len(sys.argv) > 2 else 3):
    s.run_frames(1)
    xb = s.get_x()
    inf = s.sweep_resident(True)
    dx = s.get_dx()
    sn = np.linalg.norm(dx[sv], axis=1)
    q = np.quantile(sn, [0.5, 0.9, 0.99, 1.0])
    t0 = time.perf_counter()
    cap = s.step_cap(xb, dx)
    t1 = time.perf_counter()
    print(f"frame {f}: halvings {inf['halvings']} pairs {inf['n_pairs']} |dx_sv| q50/90/99/max {q} "
          f"cap {cap:.4e} step_cap {1e3 * (t1 - t0):.2f} ms", flush=True)
