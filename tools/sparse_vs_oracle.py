"""Clustered input (BASELINE C4's mixture) on a uniform tree with empty cells: the GPU next to the
oracle's CPU restatement of the same extension (colour order).
    python tools/sparse_vs_oracle.py N DEPTH P TOL [RANK_TOL]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_1407_1572_b200 as ifmm  # noqa: E402
from oracle import ifmm_oracle as O  # noqa: E402

n, depth, p, tol = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), float(sys.argv[4])
rt = float(sys.argv[5]) if len(sys.argv) > 5 else None
X = bench.mixture_points(n)
b = np.random.default_rng(1).standard_normal(n)
tree = ifmm.build_tree(ifmm.PointSet(2, X), depth, allow_empty_leaves=True)
store = ifmm.init_operators(tree, ifmm.baseline_kernel("inv_r", n), p=p, tol=tol)
f = ifmm.factorize(store, tree, on_singular="record", rank_tol=rt)
x = ifmm.solve(f, b)
res = np.linalg.norm(ifmm.fmm_matvec(store, tree, x) - b) / np.linalg.norm(b)
rec = np.array([(r.level, r.r) for r in f.records])
t0 = time.perf_counter()
T = O.build_tree(X, depth, allow_empty=True)
spec = O.baseline_kernel("inv_r", n)
fo = O.factorize(O.init_operators(T, spec, p, tol), order="colour9", rank_tol=rt, on_singular="record")
xo = O.solve(fo, b)
t1 = time.perf_counter()
res_o = np.linalg.norm(ifmm.fmm_matvec(store, tree, xo) - b) / np.linalg.norm(b)
cnt = np.diff(tree.leaf_offsets)
print(f"mixture N={n} depth {depth} p {p} tol {tol:g} rank_tol {rt}: {int((cnt == 0).sum())} of {len(cnt)} cells empty, at most "
      f"{int(cnt.max())} points in a cell")
print(f"   GPU: residual {res:.3e} top {f.top_dim} records with unknowns {sum(1 for r in f.records if r.n + r.r > 0)} "
      f"dense kept {sum(s.fillins_dense_kept for s in f.level_stats.values())} pivots over the limit {len(f.singular_pivots)}")
print(f"   oracle (CPU, {t1 - t0:.0f} s): residual {res_o:.3e} top {int(fo.top_off[-1])} records {len(fo.recs)} dense kept "
      f"{sum(s.dense_kept for s in fo.stats.values())} pivots over the limit {len(fo.singular)}")
for k in range(depth, 1, -1):
    print(f"   level {k}: rank sum GPU {int(rec[rec[:, 0] == k, 1].sum())}  oracle {sum(r.r for r in fo.recs if r.level == k)}")
print(f"   solution GPU vs oracle {np.linalg.norm(x - xo) / np.linalg.norm(xo):.3e}", flush=True)
