import sys, time
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
from helpers import scene_inputs
from paper_2506_06494_b200.precompute_gpu import scalable_precompute
d = np.load("/root/repo/tests/golden/c1.npz"); g = {k: d[k] for k in d.files}
model, ref, h = scene_inputs(g)
for leaf in (32, 128, 512):
    t = time.time()
    pre, info = scalable_precompute(model, h, leaf_size=leaf)
    r = info["residual"]
    print(leaf, f"{time.time()-t:.2f}s", "conv", info["converged_fraction"], "median res", np.median(r), "p90", np.quantile(r, 0.9),
          "mean size", info["mean_cubature_size"], {k: round(v, 3) for k, v in info.items() if k.endswith("_s")}, flush=True)
