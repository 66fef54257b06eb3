"""Generate tests/golden/default_4k.npz from the REAL reference (build container only):
IfmmSolver() with the reference's defaults (log kernel, a = 1e-3, tol = 1e-14, p = 8,
default depth) on 4,000 seeded points in [-1, 1]^2 -- a near-exact regime with
incompressible (dense-kept) fills.  Stores b, the reference solution and residual.

Usage:  OMP_NUM_THREADS=1 OPENBLAS_NUM_THREADS=1 python oracle/gen_golden_default.py [N ...]   (4000, 8000)
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
import ifmm  # noqa: E402

OUT = os.path.join(os.path.dirname(HERE), "tests", "golden", "default_{}k.npz")


def main(n=4000):
    rng = np.random.default_rng(0)
    X = 2.0 * rng.random((n, 2)) - 1.0
    b = rng.standard_normal(n)
    est = ifmm.IfmmSolver().fit(X)
    x = est.solve(b)
    res = np.linalg.norm(est.matvec(x) - b) / np.linalg.norm(b)
    f = est.factorization_
    np.savez_compressed(OUT.format(n // 1000), n=n, b=b, x=x, resid=res, r_m=f.r_m, depth=est.tree_.depth,
                        dense_kept=sum(s.fillins_dense_kept for s in f.level_stats.values()))
    print(f"default_{n // 1000}k: residual {res:.2e} r_m {f.r_m}")


if __name__ == "__main__":
    for a in sys.argv[1:] or ["4000"]:
        main(int(a))
