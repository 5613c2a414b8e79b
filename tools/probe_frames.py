"""Diagnostic: per-frame sweep cost over a longer C4 run (profiling on/off)."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2506_06494_b200 import scenes
from paper_2506_06494_b200.local_solver import LocalSolver, SolverConfig
from paper_2506_06494_b200.model import SystemState
from paper_2506_06494_b200.precompute import Precompute

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
nframes = int(sys.argv[2]) if len(sys.argv) > 2 else 8
prof = len(sys.argv) > 3 and sys.argv[3] == "prof"
m, st, h, desc = scenes.build(name)
pre = Precompute.injected(m, h, samples=6, seed=0)
s = LocalSolver(m, SolverConfig(tol_dx=m.tol_dx, max_outer=500), precompute=pre, h_ref=h)
init = SystemState(x=st.x_prev.copy(), x_prev=st.x_prev.copy(), v=st.v.copy(), z=st.z.copy(), h=h)
s.set_frame_state(init, m.gravity)
s.profile(prof)
for f in range(nframes):
    s.phase_reset()
    rec = []
    s.timer_start()
    t0 = time.perf_counter()
    done = []
    while not done:
        done = s.run_sweeps(1, rec)
    ms = s.timer_stop()
    wall = time.perf_counter() - t0
    ph = s.phase_stats()
    n = done[0]
    print(json.dumps({"frame": f, "sweeps": n, "ms_per_sweep": round(ms / n, 2), "wall_ms_per_sweep": round(1e3 * wall / n, 2),
                      "pairs": int(np.mean([r["n_pairs"] for r in rec])), "halv": [r["halvings"] for r in rec][:8],
                      "phases": {k: round(v[0] / n, 2) for k, v in ph.items() if v[0] > 0}}), flush=True)
