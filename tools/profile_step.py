"""One assembly + factorize + solve of a bench config (for ncu launch lists / captures).

    python tools/profile_step.py [CONFIG] [rank_tol]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_1407_1572_b200 as ifmm  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3_65k"
N, kern, depth, p, tol, nrhs = bench.CONFIGS[name]
pts = 2.0 * np.random.default_rng(0).random((N, 2)) - 1.0
b = np.random.default_rng([0, 1]).standard_normal(N)
tree = ifmm.build_tree(ifmm.PointSet(2, pts), depth)
store = ifmm.init_operators(tree, ifmm.baseline_kernel(kern, N), p=p, tol=tol)
rank_tol = float(sys.argv[2]) if len(sys.argv) > 2 else None
fact = ifmm.factorize(store, tree, pivot_condition_limit=1e300, rank_tol=rank_tol)
x = ifmm.solve(fact, b)
res = np.linalg.norm(ifmm.fmm_matvec(store, tree, x) - b) / np.linalg.norm(b)
print(f"{name}: residual {res:.3e} r_m {fact.r_m} top {fact.top_dim}")
