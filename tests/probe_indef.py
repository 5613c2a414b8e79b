"""Diagnostic (not a test): per-sweep indefinite-Hessian counts on C3."""
import sys
sys.path.insert(0, ".")
from paper_2506_06494_b200 import scenes
from paper_2506_06494_b200.local_solver import LocalSolver, SolverConfig
from paper_2506_06494_b200.precompute import Precompute
m, st, h, _ = scenes.build(sys.argv[1] if len(sys.argv) > 1 else "c3")
pre = Precompute.injected(m, h)
s = LocalSolver(m, SolverConfig(), precompute=pre, h_ref=h)
s.set_state(st.x, st.z, h)
for k in range(4):
    inf = s.sweep_resident(True)
    print(k, inf["n_indefinite"], s.pre.cub_elems.size, inf["dx_norm"])
