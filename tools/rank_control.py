"""Rank-growth control (factorize(..., rank_tol=...)) against the reference-parity path:
factor + solve time, residual, rank sums, top dimension.

    python tools/rank_control.py CONFIG [rank_tol ...]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_1407_1572_b200 as ifmm  # noqa: E402

name = sys.argv[1]
tols = [None] + [float(a) for a in sys.argv[2:]]
N, kern, depth, p, tol, nrhs = bench.CONFIGS[name]
pts = 2.0 * np.random.default_rng(0).random((N, 2)) - 1.0
b = np.random.default_rng([0, 1]).standard_normal(N)
tree = ifmm.build_tree(ifmm.PointSet(2, pts), depth)
store = ifmm.init_operators(tree, ifmm.baseline_kernel(kern, N), p=p, tol=tol)
for rt in tols:
    best = None
    for rep in range(3):
        t0 = time.perf_counter()
        f = ifmm.factorize(store, tree, on_singular="record", rank_tol=rt)
        x = ifmm.solve(f, b)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
        if rep < 2:
            del f
    res = np.linalg.norm(ifmm.fmm_matvec(store, tree, x) - b) / np.linalg.norm(b)
    x1 = ifmm.solve(f, b, refine=1)
    res1 = np.linalg.norm(ifmm.fmm_matvec(store, tree, x1) - b) / np.linalg.norm(b)
    rec = np.array([(r.level, r.n, r.r) for r in f.records])
    lv = " ".join(f"L{k}: n {rec[rec[:, 0] == k, 1].mean():.0f} r {rec[rec[:, 0] == k, 2].mean():.0f}"
                  for k in range(depth, 1, -1))
    print(f"{name} rank_tol {rt}: factor+solve {best * 1e3:.1f} ms residual {res:.3e} (1 refinement step {res1:.3e}) "
          f"top {f.top_dim} rank control {f.rank_control} over-limit pivots {len(f.singular_pivots)}\n    {lv}", flush=True)
    del f
