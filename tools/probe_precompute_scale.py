"""Diagnostic: the device precompute at benchmark scale, then frames of the
scene with it (sweeps per frame, halvings)."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2506_06494_b200 import scenes
from paper_2506_06494_b200.local_solver import LocalSolver, SolverConfig
from paper_2506_06494_b200.model import SystemState
from paper_2506_06494_b200.precompute_gpu import scalable_precompute

name = sys.argv[1]
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 3
leaf = int(sys.argv[3]) if len(sys.argv) > 3 else 512
t0 = time.time()
if name.startswith("{"):  # puffer-ball variant: {"n":1,"cells":45,"youngs":[2e7],"dhat_frac":0.03,"kappa":2e3,"tank":0}
    a = json.loads(name)
    if a.get("tank"):
        m = scenes.puffer_tank(a.get("n", 10), cells=a.get("cells", 20), youngs=tuple(a.get("youngs", (2e8, 1e7))),
                               kappa=a.get("kappa", 2e3), dhat_frac=a.get("dhat_frac", 0.01))
    else:
        m = scenes.puffer_balls(a.get("n", 1), cells=a.get("cells", 45), youngs=tuple(a.get("youngs", (2e7,))),
                                kappa=a.get("kappa", 2e3), dhat_frac=a.get("dhat_frac", 0.01))
    m.tol_dx = scenes.CONTACT_TOL
    h = scenes.H
    st = scenes.predictor_state(m, SystemState.initial(m, h))
    desc = name
else:
    m, st, h, desc = scenes.build(name)
t_scene = time.time() - t0
t0 = time.time()
pre, info = scalable_precompute(m, h, leaf_size=leaf)
t_pre = time.time() - t0
res = info.pop("residual")
info.pop("converged")
print(json.dumps({"scene": desc, "ne": int(m.num_elements), "scene_s": round(t_scene, 1), "precompute_s": round(t_pre, 1),
                  "info": {k: (round(v, 4) if isinstance(v, float) else v) for k, v in info.items()},
                  "res_p50_p90": [float(np.median(res)), float(np.quantile(res, 0.9))]}), flush=True)
s = LocalSolver(m, SolverConfig(tol_dx=getattr(m, "tol_dx", 1e-3), max_outer=500), precompute=pre, h_ref=h)
init = SystemState(x=st.x_prev.copy(), x_prev=st.x_prev.copy(), v=st.v.copy(), z=st.z.copy(), h=h)
s.set_frame_state(init, m.gravity)
for f in range(frames):
    rec = []
    t0 = time.time()
    done = []
    while not done:
        done = s.run_sweeps(1, rec)
    hv = [r["halvings"] for r in rec]
    print(json.dumps({"frame": f, "sweeps": done[0], "s": round(time.time() - t0, 2), "halvings": hv[:20],
                      "le5": float(np.mean(np.array(hv) <= 5))}), flush=True)
