"""Robustness sweep of the public API over reference-style parameters
(IfmmSolver defaults: log kernel, a = 1e-3, tol = 1e-14, p = 8; other registry
kernels; 1-D / 3-D).  Prints residual vs the store's FMM operator or the error."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1407_1572_b200 as ifmm  # noqa: E402

CASES = [
    # (dim, N, kernel, a, tol, p, depth or None)
    (2, 1000, "log", 1e-3, 1e-14, 8, None),
    (2, 2000, "log", 1e-3, 1e-14, 8, None),
    (2, 4000, "log", 1e-3, 1e-14, 8, None),
    (2, 8000, "log", 1e-3, 1e-14, 8, None),
    (2, 16000, "log", 1e-3, 1e-14, 8, None),
    (2, 4000, "log", 1e-3, 1e-10, 6, None),
    (2, 4000, "gaussian", 1e-3, 1e-10, 6, None),
    (2, 4000, "multiquadric", 1e-3, 1e-10, 6, None),
    (2, 4000, "inverse-multiquadric", 1e-3, 1e-10, 6, None),
    (2, 4000, "inverse-quadric", 1e-3, 1e-10, 6, None),
    (2, 4000, "helmholtz3d", 1e-3, 1e-10, 6, None),
    (2, 4000, "bessel-y0", 1e-3, 1e-10, 6, None),
    (2, 4000, "biharmonic", 1e-3, 1e-10, 6, None),
    (2, 16384, "log", 1e-3, 1e-8, 4, 4),
    (2, 16384, "log", 1e-3, 1e-8, 4, 5),
    (1, 2000, "log", 1e-3, 1e-12, 8, None),
    (3, 4000, "laplace3d", 1e-3, 1e-8, 4, 2),
    (3, 8000, "laplace3d", 1e-3, 1e-6, 3, 3),
]
for dim, n, kern, a, tol, p, depth in CASES:
    rng = np.random.default_rng(0)
    X = 2.0 * rng.random((n, dim)) - 1.0
    b = rng.standard_normal(n)
    t0 = time.perf_counter()
    try:
        est = ifmm.IfmmSolver(kernel=kern, a=a, tol=tol, p=p, depth=depth).fit(X)
        x = est.solve(b)
        res = np.linalg.norm(est.matvec(x) - b) / np.linalg.norm(b)
        f = est.factorization_
        print(f"dim={dim} N={n} {kern} tol={tol:g} p={p} depth={est.tree_.depth}: residual {res:.2e} r_m {f.r_m} "
              f"top {f.top_dim} dense_kept {sum(s.fillins_dense_kept for s in f.level_stats.values())} "
              f"({time.perf_counter() - t0:.2f} s)", flush=True)
    except Exception as e:
        print(f"dim={dim} N={n} {kern} tol={tol:g} p={p} depth={depth}: FAILED {type(e).__name__}: {e}", flush=True)
