"""Diagnostic: the reference's cube_drop scene with the reference's own
precompute vs the device precompute (same frames, activations per sweep)."""
import sys
import numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from helpers import scene_inputs
from paper_2506_06494_b200.local_solver import LocalSolver, SolverConfig
from paper_2506_06494_b200.model import SystemState
from paper_2506_06494_b200.precompute_gpu import scalable_precompute
name = sys.argv[1] if len(sys.argv) > 1 else "cube_drop"
d = np.load(f"tests/golden/{name}.npz"); g = {k: d[k] for k in d.files}
model, ref, h = scene_inputs(g)
c = g["scene_cfg"]
for label, pre in (("reference", ref), ("device", scalable_precompute(model, h, leaf_size=int(sys.argv[2]) if len(sys.argv) > 2 else 512)[0])):
    s = LocalSolver(model, SolverConfig(tol_dx=float(c[0]), max_outer=int(c[1])), precompute=pre, h_ref=h)
    st = SystemState.initial(model, h)
    s.set_frame_state(st, model.gravity)
    its, acts = [], []
    for f in range(g["frame_iterations"].size):
        rec = []
        done = []
        while not done:
            done = s.run_sweeps(1, rec)
        its.append(done[0]); acts += [r["halvings"] for r in rec]
    xp, _ = s.get_frame_state()
    print(label, "sweeps/frame", its, "\n  halvings", acts[:60], "\n  ymin", float(xp[:, 1].min()), flush=True)
