"""Debug: residual of repeated factorizations on one store (workspace reuse check)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_1407_1572_b200 as ifmm  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3_262k"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
N, kern, depth, p, tol, nrhs = bench.CONFIGS[name]
pts = 2.0 * np.random.default_rng(0).random((N, 2)) - 1.0
b = np.random.default_rng([0, 1]).standard_normal(N)
tree = ifmm.build_tree(ifmm.PointSet(2, pts), depth)
store = ifmm.init_operators(tree, ifmm.baseline_kernel(kern, N), p=p, tol=tol)
for it in range(reps):
    fact = ifmm.factorize(store, tree, pivot_condition_limit=1e15)
    x = ifmm.solve(fact, b)
    res = np.linalg.norm(ifmm.fmm_matvec(store, tree, x) - b) / np.linalg.norm(b)
    print(f"{name} rep {it}: residual {res:.3e} r_m {fact.r_m} top {fact.top_dim} ms {fact.factor_ms:.1f}", flush=True)
    print("   level stats:", {k: (s.max_rank, s.fillins_compressed, s.fillins_dense_kept)
                              for k, s in fact.level_stats.items()}, flush=True)
    x2 = ifmm.solve(fact, b, refine=6, target=1e-9)
    print("   refinement history:", ["%.2e" % v for v in fact.last_refinement], flush=True)
    del fact
