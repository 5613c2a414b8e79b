"""Diagnostic (not a test): contact statistics of a scene's first sweeps."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2506_06494_b200 import scenes
from paper_2506_06494_b200.local_solver import LocalSolver, SolverConfig
from paper_2506_06494_b200.precompute import Precompute
name = sys.argv[1] if len(sys.argv) > 1 else "c4"
m, st, h, d = scenes.build(name)
print(d, m.num_vertices, len(m.surface_vertices), len(m.surface_tris), "dhat", m.barrier.dhat, flush=True)
pre = Precompute.injected(m, h, neighbor_scale=float(sys.argv[3]) if len(sys.argv) > 3 else 0.6)
s = LocalSolver(m, SolverConfig(tol_dx=getattr(m, "tol_dx", 1e-3)), precompute=pre, h_ref=h)
for label, x in (("x0", m.initial_positions), ("z", st.z)):
    p = s.find_pairs(x)
    for k in (0, 1):
        sel = p[p[:, 0] == k]
        print(label, "kind", k, "n", len(sel), "min d", sel[:, 6].min() if len(sel) else None, flush=True)
from paper_2506_06494_b200.model import SystemState
init = SystemState(x=st.x_prev.copy(), x_prev=st.x_prev.copy(), v=st.v.copy(), z=st.z.copy(), h=h)
s.set_frame_state(init, m.gravity)
for f in range(int(sys.argv[2]) if len(sys.argv) > 2 else 4):
    try:
        done = s.run_frames(1)
    except Exception as exc:
        print("frame sweep", f, "failed:", exc)
        break
    x = s.get_x()
    print("sweep", f, done, "finite", bool(np.isfinite(x).all()), "ymin", x[:, 1].min(), flush=True)
s.set_state(st.x, st.z, h)
for it in range(6):
    xb = s.get_x()
    try:
        inf = s.sweep_resident(True)
    except Exception as exc:
        print("sweep", it, "failed:", exc)
        p = s.find_pairs(xb)
        print("pairs at start", len(p), "min d", p[:, 6].min())
        break
    print("sweep", it, {k: inf[k] for k in ("n_pairs", "halvings", "dx_norm", "max_local_step",
                                            "line_search_activations", "energy")}, flush=True)
