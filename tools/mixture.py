"""Experiment (IFMM_EXPERIMENTAL_EMPTY_LEAVES=1): clustered inputs (BASELINE C4s 16-component Gaussian mixture, std 0.05, clipped to [0,1]^2,
duplicates redrawn) on a uniform tree with empty leaf cells; residual vs the FMM operator and,
for small N, the solution vs dense LU.

    python tools/mixture.py N DEPTH P TOL
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1407_1572_b200 as ifmm  # noqa: E402
from oracle import ifmm_oracle as O  # noqa: E402


def mixture_points(n, seed=0, comps=16, std=0.05):
    rng = np.random.default_rng(seed)
    means = rng.random((comps, 2))
    pts = np.empty((0, 2))
    while len(pts) < n:
        c = rng.integers(0, comps, n)
        x = np.clip(means[c] + std * rng.standard_normal((n, 2)), 0.0, 1.0)
        pts = np.unique(np.concatenate([pts, x]), axis=0)
    pts = pts[rng.permutation(len(pts))[:n]]
    return 2.0 * pts - 1.0


n, depth, p, tol = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), float(sys.argv[4])
X = mixture_points(n)
kern = ifmm.baseline_kernel("inv_r", n)
tree = ifmm.build_tree(ifmm.PointSet(2, X), depth)
cnt = np.diff(tree.leaf_offsets)
print(f"N={n} depth={depth}: {len(cnt)} leaves, {int((cnt == 0).sum())} empty, max {int(cnt.max())} points")
store = ifmm.init_operators(tree, kern, p=p, tol=tol)
f = ifmm.factorize(store, tree)
b = np.random.default_rng(1).standard_normal(n)
x = ifmm.solve(f, b)
res = np.linalg.norm(ifmm.fmm_matvec(store, tree, x) - b) / np.linalg.norm(b)
print(f"residual vs FMM operator {res:.3e}, r_m {f.r_m}, top {f.top_dim}")
if n <= 8192:
    A = O.dense_matrix(O.baseline_kernel("inv_r", n), X)
    xd = np.linalg.solve(A, b)
    print(f"vs dense LU: {np.linalg.norm(x - xd) / np.linalg.norm(xd):.3e}")
