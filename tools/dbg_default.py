"""Debug: reference-default config (log, a=1e-3, tol=1e-14, p=8) on the GPU vs the oracle (colour9)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1407_1572_b200 as ifmm  # noqa: E402
from oracle import ifmm_oracle as O  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4000
rng = np.random.default_rng(0)
X = 2.0 * rng.random((n, 2)) - 1.0
b = rng.standard_normal(n)
depth = ifmm.default_depth(n, 2)
tree = ifmm.build_tree(ifmm.PointSet(2, X), depth)
kern = ifmm.make_kernel("log", a=1e-3)
store = ifmm.init_operators(tree, kern, p=8, tol=1e-14)
for k in range(2, depth + 1):
    n_, r_ = store._level_dims(k)
    print(f"level {k}: n min/mean/max {n_.min()}/{n_.mean():.1f}/{n_.max()}  r0 min/mean/max {r_.min()}/{r_.mean():.1f}/{r_.max()}"
          f"  r0>n: {(r_ > n_).sum()}")
f = ifmm.factorize(store, tree, pivot_condition_limit=1e300)
x = ifmm.solve(f, b)
res = np.linalg.norm(ifmm.fmm_matvec(store, tree, x) - b) / np.linalg.norm(b)
print("gpu stats", {k: (s.max_rank, s.fillins_compressed, s.fillins_dense_kept) for k, s in f.level_stats.items()},
      "top", f.top_dim, "resid", res)
T = O.build_tree(X, depth)
st = O.init_operators(T, O.KernelSpec("log", a=1e-3), 8, 1e-14)
fo = O.factorize(st, order="colour9")
print("oracle stats", {k: (s.max_rank, s.compressed, s.dense_kept) for k, s in fo.stats.items()} if hasattr(fo, "stats") else vars(fo).keys())
