"""Clustered inputs (BASELINE C4s 16-component Gaussian mixture, std 0.05, clipped to [0,1]^2,
duplicates redrawn) on a uniform tree with empty leaf cells; residual vs the FMM operator and,
for small N, the solution vs dense LU.

    python tools/mixture.py N DEPTH P TOL [RANK_TOL]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1407_1572_b200 as ifmm  # noqa: E402
from oracle import ifmm_oracle as O  # noqa: E402


from bench import mixture_points  # noqa: E402

n, depth, p, tol = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), float(sys.argv[4])
X = mixture_points(n)
kern = ifmm.baseline_kernel("inv_r", n)
rank_tol = float(sys.argv[5]) if len(sys.argv) > 5 else None
tree = ifmm.build_tree(ifmm.PointSet(2, X), depth, allow_empty_leaves=True)
cnt = np.diff(tree.leaf_offsets)
print(f"N={n} depth={depth}: {len(cnt)} leaves, {int((cnt == 0).sum())} empty, max {int(cnt.max())} points")
store = ifmm.init_operators(tree, kern, p=p, tol=tol)
import time  # noqa: E402
t0 = time.perf_counter()
f = ifmm.factorize(store, tree, on_singular="record", rank_tol=rank_tol)
print(f"factorize {time.perf_counter() - t0:.2f} s, rank control {f.rank_control}, pivots over the limit "
      f"{len(f.singular_pivots)}, max cond {max(f.max_cond.values()):.2e}")
b = np.random.default_rng(1).standard_normal(n)
x = ifmm.solve(f, b)
res = np.linalg.norm(ifmm.fmm_matvec(store, tree, x) - b) / np.linalg.norm(b)
print(f"residual vs FMM operator {res:.3e}, r_m {f.r_m}, top {f.top_dim}")
if n <= 8192:
    A = O.dense_matrix(O.baseline_kernel("inv_r", n), X)
    xd = np.linalg.solve(A, b)
    print(f"vs dense LU: {np.linalg.norm(x - xd) / np.linalg.norm(xd):.3e}")
