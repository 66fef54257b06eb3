"""Rank-growth control over the reference's kernel registry (ifmm/kernels.py:160-170) through
IfmmSolver: residual and rank sums with and without rank_tol.
    python tools/rank_control_registry.py [N] [tol] [rank_tol]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1407_1572_b200 as ifmm  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 16000
tol = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-6
rt = float(sys.argv[3]) if len(sys.argv) > 3 else tol / 10
rng = np.random.default_rng(0)
X = rng.uniform(-1, 1, (N, 2))
b = rng.standard_normal(N)
for name in ["log", "laplace3d", "biharmonic", "bessel-y0", "inverse-quadric", "inverse-multiquadric", "helmholtz3d",
             "gaussian", "multiquadric"]:
    out = []
    for r in (None, rt):
        try:
            est = ifmm.IfmmSolver(kernel=name, a=1e-3, tol=tol, p=6, rank_tol=r).fit(X)
            x = est.solve(b)
            res = np.linalg.norm(est.matvec(x) - b) / np.linalg.norm(b)
            rs = sum(q.r for q in est.factorization_.records)
            out.append(f"residual {res:.2e} rank sum {rs} top {est.factorization_.top_dim}")
        except Exception as e:  # noqa: BLE001
            out.append(f"{type(e).__name__}: {str(e)[:60]}")
    print(f"{name:22s} parity: {out[0]}   rank_tol {rt:g}: {out[1]}", flush=True)
