"""Scale parity fixtures: the CPU oracle (oracle/jgs2_oracle.py, itself pinned
to the reference's goldens by tests/test_oracle_golden.py) run on
scaled-down BASELINE constructions, frame by frame like harness.run
(harness.py:187-211): compute_z, capped initialize_step, outer_solve to
tol_dx, velocity update. Run once in the build container:

    python tests/golden/make_scale_goldens.py [name ...]

Inputs are regenerated deterministically on the GPU box (scenes.build +
Precompute.injected(seed 0)), so a fixture stores only outputs: per frame
the final positions and iteration count, per sweep the halvings, dx norm,
energy and accepted gamma. The vertex-triangle narrowphase uses the oracle's
exact spatial pruning (identical pair sets, tests/test_oracle_golden.py)."""

import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import jgs2_oracle as orc  # noqa: E402
from paper_2506_06494_b200 import scenes  # noqa: E402
from paper_2506_06494_b200.model import SystemState  # noqa: E402
from paper_2506_06494_b200.precompute import Precompute  # noqa: E402

# name -> frames (C4 tank >= 12 cells/ball; the touching tank for v-t pairs;
# C3 at half resolution; C2 at 20 cells)
CASES = {"c4s12": 3, "c4t8": 2, "c3s2": 3, "c2s20": 3}


def run(name, frames):
    t0 = time.time()
    orc.PRUNE = True
    m, st0, h, desc = scenes.build(name)
    pre = Precompute.injected(m, h, samples=6, seed=0)
    cfg = orc.OracleConfig(tol_dx=getattr(m, "tol_dx", 1e-3), max_outer=500)
    S = orc.OracleSolver(m, pre, h, cfg)
    st = SystemState.initial(m, h)
    out = {"frame_x_final": [], "frame_iterations": [], "frame_cap": [], "sweep_frame": [],
           "sweep_halvings": [], "sweep_dx_norm": [], "sweep_energy": [], "sweep_x": []}
    for f in range(frames):
        st.z = orc.compute_z(m, st.x_prev, st.v, h)
        dz = st.z - st.x_prev
        cap = orc.feasibility_cap(m, st.x_prev, dz) if (m.barrier is not None) else 1.0
        st.x = st.x_prev + cap * dz
        out["frame_cap"].append(cap)
        for it in range(cfg.max_outer):
            rot = orc.vertex_rotations(m, st.x)
            dx, info = S.sweep(st, rot)
            dxn = float(m.normalization.scale * np.linalg.norm(dx))
            acts = info["line_search_activations"]
            out["sweep_frame"].append(f)
            out["sweep_halvings"].append(acts)
            out["sweep_dx_norm"].append(dxn)
            out["sweep_energy"].append(orc.total_energy(m, st.z, h, st.x, orc.find_pairs(m, st.x)))
            if f == 0 and it < 2:
                out["sweep_x"].append(st.x.copy())
            if dxn < cfg.tol_dx:
                break
        out["frame_iterations"].append(it + 1)
        out["frame_x_final"].append(st.x.copy())
        st.v = (st.x - st.x_prev) / h
        st.x_prev = st.x.copy()
        print(f"{name} frame {f}: {it + 1} sweeps, halvings {out['sweep_halvings'][-(it + 1):][:12]}, "
              f"{time.time() - t0:.0f}s", flush=True)
    import scipy
    np.savez_compressed(Path(__file__).parent / f"scale_{name}.npz",
                        scene=np.array([name]), h=np.array([h]), tol_dx=np.array([cfg.tol_dx]),
                        nv=np.array([m.num_vertices]), ne=np.array([m.num_elements]),
                        meta_versions=np.array([np.__version__, scipy.__version__]),
                        **{k: np.asarray(v) for k, v in out.items()})


if __name__ == "__main__":
    for name in sys.argv[1:] or CASES:
        run(name, CASES.get(name, 2))
