"""FLOP rates of the per-batch GEMM phases from a timed factorization.

    python tools/xgemm_rate.py [CONFIG]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_1407_1572_b200 as ifmm  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
N, kern, depth, p, tol, nrhs = bench.CONFIGS[name]
pts = 2.0 * np.random.default_rng(0).random((N, 2)) - 1.0
tree = ifmm.build_tree(ifmm.PointSet(2, pts), depth)
store = ifmm.init_operators(tree, ifmm.baseline_kernel(kern, N), p=p, tol=tol)
f = ifmm.factorize(store, tree, pivot_condition_limit=1e15)
del f
f = ifmm.factorize(store, tree, pivot_condition_limit=1e15, timing=True)
recs = f.records
by = {}
for R in recs:
    m = R.n + R.r
    d = by.setdefault(R.level, [0.0, 0.0, 0, 0.0])
    d[0] += 2.0 * m * R.n * (R.w - R.r)   # X = S^-1(:, :n) C
    d[1] += 2.0 * m ** 3                  # Gauss-Jordan
    d[2] += 1
    d[3] += R.n * float(R.w - R.r) * (R.w - R.r + 1) + 2.0 * R.n * (R.w - R.r) * R.r  # Schur, ~upper triangle
lv = f.phase_times_by_level
for k in sorted(by, reverse=True):
    x, gj, cnt, sc = by[k]
    t = lv.get(k, {})
    print(f"level {k}: {cnt:6d} pivots  X {x / 1e12:.3f} TF in {t.get('x_gemm', 0):.1f} ms = "
          f"{x / max(1e-9, t.get('x_gemm', 0)) / 1e9:.1f} TF/s | GJ {gj / 1e12:.3f} TF in "
          f"{t.get('gauss_jordan', 0):.1f} ms = {gj / max(1e-9, t.get('gauss_jordan', 0)) / 1e9:.1f} TF/s | Schur "
          f"~{sc / 1e12:.3f} TF in {t.get('schur_gemm', 0):.1f} ms = "
          f"{sc / max(1e-9, t.get('schur_gemm', 0)) / 1e9:.1f} TF/s")
