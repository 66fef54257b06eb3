"""GPU factorize+solve of a golden case vs the reference's results stored in tests/golden."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1407_1572_b200 as ifmm  # noqa: E402
from oracle import ifmm_oracle as O  # noqa: E402

for name in sys.argv[1:]:
    g = dict(np.load(os.path.join(ROOT, "tests", "golden", f"{name}.npz")))
    N, depth = int(g["N"]), int(g["depth"])
    pts = O.baseline_points(N, seed=0)
    tree = ifmm.build_tree(ifmm.PointSet(2, pts), depth)
    kern = ifmm.make_kernel(str(g["kernel"]), a=float(g["a"]), scale=float(g["scale"]), shift=float(g["shift"]))
    store = ifmm.init_operators(tree, kern, p=int(g["p"]), tol=float(g["tol"]))
    f = ifmm.factorize(store, tree)
    x = ifmm.solve(f, g["b"])
    b = g["b"]
    res = np.linalg.norm(ifmm.fmm_matvec(store, tree, x) - b) / np.linalg.norm(b)
    xc, xm = g["x_colour9"], g["x_morton"]
    rel = lambda a, c: np.linalg.norm(a - c) / np.linalg.norm(c)
    print(f"{name}: residual gpu {res:.2e} | reference Morton {float(g['resid_morton']):.2e} colour9 "
          f"{float(g['resid_colour9']):.2e} | x vs ref colour9 {rel(x, xc):.2e}, vs ref Morton {rel(x, xm):.2e}, "
          f"ref Morton vs colour9 {rel(xm, xc):.2e} | r_m {f.r_m} (ref {int(g['rm_morton'])}/{int(g['rm_colour9'])}) "
          f"top {f.top_dim} (ref {int(g['top_morton'])}/{int(g['top_colour9'])})", flush=True)
