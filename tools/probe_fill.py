import sys; sys.path.insert(0, "/root/repo")
from paper_2506_06494_b200 import scenes
from paper_2506_06494_b200.local_solver import LocalSolver, SolverConfig
from paper_2506_06494_b200.precompute import Precompute
for name in sys.argv[1:]:
    m, st, h, d = scenes.build(name)
    s = LocalSolver(m, SolverConfig(), precompute=Precompute.injected(m, h), h_ref=h)
    a, b, c = s.factor_fill()
    print(name, "stored", a, "nd exact", b, "metis exact", c, "nd/metis", b / c, "stored/metis", a / c, flush=True)
