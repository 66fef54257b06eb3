"""IfmmSolver() defaults (log, a=1e-3, tol=1e-14, p=8) on N seeded points: per-level
max pivot condition, dense-kept fills, residual and solution vs the reference golden."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1407_1572_b200 as ifmm  # noqa: E402

for name in sys.argv[1:]:
    g = dict(np.load(os.path.join(ROOT, "tests", "golden", f"{name}.npz")))
    n = int(g["n"])
    X = 2.0 * np.random.default_rng(0).random((n, 2)) - 1.0
    tree = ifmm.build_tree(ifmm.PointSet(2, X), int(g["depth"]))
    store = ifmm.init_operators(tree, ifmm.make_kernel("log", a=1e-3), p=8, tol=1e-14)
    f = ifmm.factorize(store, tree, on_singular="record")
    x = ifmm.solve(f, g["b"])
    res = np.linalg.norm(ifmm.fmm_matvec(store, tree, x) - g["b"]) / np.linalg.norm(g["b"])
    print(f"{name}: residual {res:.2e} (ref {float(g['resid']):.2e}) x diff {np.linalg.norm(x - g['x']) / np.linalg.norm(g['x']):.2e}"
          f" r_m {f.r_m} (ref {int(g['r_m'])}) top {f.top_dim}")
    for k in sorted(f.level_stats):
        s = f.level_stats[k]
        print(f"  level {k}: max cond {f.max_cond[k]:.2e} max rank {s.max_rank} compressed {s.fillins_compressed} "
              f"dense kept {s.fillins_dense_kept}")
    R = np.array([(r.level, r.index, r.n, r.r, r.w) for r in f.records])
    for k in sorted(set(R[:, 0])):
        q = R[R[:, 0] == k]
        print(f"  level {k}: n {q[:, 2].min()}..{q[:, 2].max()} r {q[:, 3].min()}..{q[:, 3].max()} w max {q[:, 4].max()}")
    print("  singular:", f.singular_pivots[:8], flush=True)
