"""Diagnostic: per-sweep device time and phase breakdown; the slowest sweeps."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2506_06494_b200 import scenes
from paper_2506_06494_b200.local_solver import LocalSolver, SolverConfig
from paper_2506_06494_b200.model import SystemState
from paper_2506_06494_b200.precompute import Precompute

m, st, h, desc = scenes.build(sys.argv[1] if len(sys.argv) > 1 else "c4")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 300
pre = Precompute.injected(m, h, samples=6, seed=0)
s = LocalSolver(m, SolverConfig(tol_dx=m.tol_dx, max_outer=500), precompute=pre, h_ref=h)
init = SystemState(x=st.x_prev.copy(), x_prev=st.x_prev.copy(), v=st.v.copy(), z=st.z.copy(), h=h)
s.set_frame_state(init, m.gravity)
s.profile(True)
rows = []
for k in range(n):
    s.phase_reset()
    rec = []
    t0 = time.perf_counter()
    s.timer_start()
    s.run_sweeps(1, rec)
    ms = s.timer_stop()
    wall = 1e3 * (time.perf_counter() - t0)
    ph = s.phase_stats()
    rows.append((ms, wall, k, rec[0]["halvings"], rec[0]["n_pairs"], {p: round(v[0], 2) for p, v in ph.items() if v[0] > 0.3}))
ms = np.array([r[0] for r in rows])
print("median", np.median(ms), "mean", ms.mean(), "p90", np.quantile(ms, 0.9), "max", ms.max())
for r in sorted(rows, key=lambda r: -r[0])[:12]:
    print(json.dumps({"ms": round(r[0], 2), "wall": round(r[1], 2), "sweep": r[2], "halv": r[3], "pairs": r[4], "ph": r[5]}))
