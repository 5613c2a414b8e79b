"""Diagnostic (not a test): backtracking behaviour of contact-scene variants
on the device. Prints per-frame sweeps and the halvings histogram."""
import json
import sys
import time
import numpy as np
sys.path.insert(0, ".")
from paper_2506_06494_b200 import scenes
from paper_2506_06494_b200.local_solver import LocalSolver, SolverConfig
from paper_2506_06494_b200.precompute import Precompute
from paper_2506_06494_b200.model import SystemState


def run(cells, youngs, kappa, dhat_frac, frames, tol, max_outer=100, ws=0.05, n=10, walls=None, ncols=4, mode="jacobi", sg=0.5, so=0.0, tank=False, bg=4.0):
    t0 = time.time()
    m = scenes.puffer_tank(n, cells=cells, youngs=youngs, kappa=kappa, dhat_frac=dhat_frac, ball_gap=bg) if tank else scenes.puffer_balls(n, cells=cells, youngs=youngs, walls=(n > 1) if walls is None else walls, kappa=kappa, dhat_frac=dhat_frac, ncols=ncols, stack_gap=sg, stack_offset=so)
    h = scenes.H
    pre = Precompute.injected(m, h, weight_scale=ws)
    s = LocalSolver(m, SolverConfig(tol_dx=tol, max_outer=max_outer, mode=mode), precompute=pre, h_ref=h)
    st = SystemState.initial(m, h)
    s.set_frame_state(st, m.gravity)
    hist = np.zeros(33, dtype=int)
    per_frame = []
    from paper_2506_06494_b200 import _lib as L
    cap = L.f64(1.0)
    import ctypes
    for f in range(frames):
        s._call(s._lib.jgs2_frame_begin, ctypes.byref(cap))
        it = 0
        hs = []
        for it in range(1, max_outer + 1):
            inf = s.sweep_resident(True)
            hs.append(int(inf["halvings"]))
            hist[min(inf["halvings"], 32)] += 1
            if inf["dx_norm"] < tol:
                break
        s._call(s._lib.jgs2_frame_end)
        xp, _ = s.get_frame_state()
        per_frame.append((int(it), round(float(cap.value), 4), round(float(xp[:, 1].min()) / m.barrier.dhat, 4), hs[:10]))
    xp, v = s.get_frame_state()
    ymin = float(xp[:, 1].min())
    nsw = hist.sum()
    good = hist[:6].sum() / max(nsw, 1)
    print(json.dumps({"n": n, "walls": walls, "ncols": ncols, "mode": mode, "sg": sg, "so": so, "tank": tank, "bg": bg, "cells": cells, "youngs": youngs, "kappa": kappa, "dhat_frac": dhat_frac, "tol": tol, "ws": ws,
                      "ne": int(m.num_elements), "sweeps": int(nsw), "frac_le5": round(float(good), 3),
                      "floored": int(hist[31:].sum()),
                      "frames": per_frame, "secs": round(time.time() - t0, 1)}), flush=True)


if __name__ == "__main__":
    for spec in sys.argv[1:]:
        a = json.loads(spec)
        run(a.get("cells", 20), tuple(a.get("youngs", (1e6, 5e4))), a.get("kappa", 2e3), a.get("dhat_frac", 0.01),
            a.get("frames", 6), a.get("tol", 2.5e-5), a.get("max_outer", 60), a.get("ws", 0.05), a.get("n", 10), a.get("walls"), a.get("ncols", 4), a.get("mode", "jacobi"), a.get("sg", 0.5), a.get("so", 0.0), a.get("tank", False), a.get("bg", 4.0))
