"""Debug: compare GPU elimination records (n, r, w) and level stats with the oracle."""
import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_1407_1572_b200 as ifmm
from oracle import ifmm_oracle as O
from conftest import load_golden, golden_kernel
name = sys.argv[1] if len(sys.argv) > 1 else "reglog_1k"
g = load_golden(name)
N, depth, p, tol = int(g["N"]), int(g["depth"]), int(g["p"]), float(g["tol"])
pts = O.baseline_points(N, 0)
k = ifmm.make_kernel(str(g["kernel"]), a=float(g["a"]), scale=float(g["scale"]), shift=float(g["shift"]))
tree = ifmm.build_tree(ifmm.PointSet(2, pts), depth)
store = ifmm.init_operators(tree, k, p=p, tol=tol)
f = ifmm.factorize(store, tree)
recs = f.records
T = O.build_tree(pts, depth)
so = O.init_operators(T, golden_kernel(g), p, tol)
fo = O.factorize(so, order="colour9")
print("gpu r_m", f.r_m, "top", f.top_dim, {kk: vars(v) for kk, v in f.level_stats.items()})
print("ora r_m", fo.r_m, "top", int(fo.top_off[-1]), {kk: (v.clusters, v.max_rank, v.compressed, v.dense_kept) for kk, v in fo.stats.items()})
nd = 0
for a, b in zip(recs, fo.recs):
    wo = sum(so.n(b.level, j) for j in b.xp) + sum(so.r(b.level, j) for j in b.yp) + b.r
    if (a.level, a.index, a.n, a.r) != (b.level, b.index, b.n, b.r) or nd < 5:
        print("gpu", (a.level, a.index, a.n, a.r, a.w), "ora", (b.level, b.index, b.n, b.r, wo, len(b.xp), len(b.yp)))
        nd += 1
    if nd > 30: break
