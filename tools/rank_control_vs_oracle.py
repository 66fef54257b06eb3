"""Rank-growth control at a larger size: the GPU (factorize(..., rank_tol=)) next to the oracle's CPU
restatement of the same procedure (oracle/ifmm_oracle.py::_consolidate, colour order).
    python tools/rank_control_vs_oracle.py CONFIG RANK_TOL        (e.g. C3_262k 1e-7: ~6 min of one core)"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_1407_1572_b200 as ifmm  # noqa: E402
from oracle import ifmm_oracle as O  # noqa: E402

name, rt = sys.argv[1], float(sys.argv[2])
N, kern, depth, p, tol, _ = bench.CONFIGS[name]
pts = O.baseline_points(N, seed=0)
b = O.baseline_rhs(N, "normal")
tree = ifmm.build_tree(ifmm.PointSet(2, pts), depth)
store = ifmm.init_operators(tree, ifmm.baseline_kernel(kern, N), p=p, tol=tol)
f = ifmm.factorize(store, tree, on_singular="record", rank_tol=rt)
x = ifmm.solve(f, b)
res = np.linalg.norm(ifmm.fmm_matvec(store, tree, x) - b) / np.linalg.norm(b)
rec = np.array([(r.level, r.r) for r in f.records])
t0 = time.perf_counter()
T = O.build_tree(pts, depth)
spec = O.baseline_kernel(kern, N)
fo = O.factorize(O.init_operators(T, spec, p, tol), order="colour9", rank_tol=rt, on_singular="record")
xo = O.solve(fo, b)
t1 = time.perf_counter()
res_o = np.linalg.norm(ifmm.fmm_matvec(store, tree, xo) - b) / np.linalg.norm(b)
print(f"{name} rank_tol {rt:g}: GPU residual {res:.3e} top {f.top_dim} rank control {f.rank_control} pivots over the limit "
      f"{len(f.singular_pivots)}")
print(f"   oracle (CPU, {t1 - t0:.0f} s): residual {res_o:.3e} top {int(fo.top_off[-1])} rank control {tuple(fo.rank_control)} "
      f"pivots over the limit {len(fo.singular)}")
for k in range(depth, 1, -1):
    print(f"   level {k}: rank sum GPU {int(rec[rec[:, 0] == k, 1].sum())}  oracle {sum(r.r for r in fo.recs if r.level == k)}")
print(f"   solution GPU vs oracle {np.linalg.norm(x - xo) / np.linalg.norm(xo):.3e}", flush=True)
