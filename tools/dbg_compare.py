"""Debug: GPU vs oracle (colour9) level statistics and residual for one configuration.

    python tools/dbg_compare.py KERNEL N DEPTH P TOL [A]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1407_1572_b200 as ifmm  # noqa: E402
from oracle import ifmm_oracle as O  # noqa: E402

kern, n, depth, p, tol = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), float(sys.argv[5])
a = float(sys.argv[6]) if len(sys.argv) > 6 else 1e-3
rng = np.random.default_rng(0)
X = 2.0 * rng.random((n, 2)) - 1.0
b = rng.standard_normal(n)
tree = ifmm.build_tree(ifmm.PointSet(2, X), depth)
store = ifmm.init_operators(tree, ifmm.make_kernel(kern, a=a), p=p, tol=tol)
f = ifmm.factorize(store, tree, pivot_condition_limit=1e300)
x = ifmm.solve(f, b)
res = np.linalg.norm(ifmm.fmm_matvec(store, tree, x) - b) / np.linalg.norm(b)
print("gpu   ", {k: (s.max_rank, s.fillins_compressed, s.fillins_dense_kept) for k, s in sorted(f.level_stats.items())},
      f"top {f.top_dim} resid {res:.3e}", flush=True)
T = O.build_tree(X, depth)
st = O.init_operators(T, O.KernelSpec(kern, a=a), p, tol)
fo = O.factorize(st, order="colour9")
xo = O.solve(fo, b)
st2 = O.init_operators(T, O.KernelSpec(kern, a=a), p, tol)
reso = np.linalg.norm(O.fmm_matvec(st2, xo) - b) / np.linalg.norm(b)
print("oracle", {k: (s.max_rank, s.compressed, s.dense_kept) for k, s in sorted(fo.stats.items())},
      f"resid {reso:.3e} diff {np.linalg.norm(x - xo) / np.linalg.norm(xo):.3e}", flush=True)
