"""Per-level comparison of a GPU factorization with a reference golden run:
final rank sums, largest pivot condition estimate, compressed fills, the
pivots over the 1e12 limit, residual and solution differences.

    python tools/diag_levels.py c3_262k [c3_1m ...]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1407_1572_b200 as ifmm  # noqa: E402
from oracle import ifmm_oracle as O  # noqa: E402

for name in sys.argv[1:]:
    g = dict(np.load(os.path.join(ROOT, "tests", "golden", f"{name}.npz")))
    N, depth, p, tol = int(g["N"]), int(g["depth"]), int(g["p"]), float(g["tol"])
    pts = O.baseline_points(N, seed=0)
    tree = ifmm.build_tree(ifmm.PointSet(2, pts), depth)
    kname = str(g["kernel"])
    if "scale" in g:
        kern = ifmm.make_kernel(kname, a=float(g["a"]), scale=float(g["scale"]), shift=float(g["shift"]))
    else:
        kern = ifmm.baseline_kernel(kname, N)
    store = ifmm.init_operators(tree, kern, p=p, tol=tol)
    t0 = time.perf_counter()
    f = ifmm.factorize(store, tree, on_singular="record")
    t1 = time.perf_counter()
    b = g["b"] if "b" in g else O.baseline_rhs(N, "normal")
    x = ifmm.solve(f, b)
    res = np.linalg.norm(ifmm.fmm_matvec(store, tree, x) - b) / np.linalg.norm(b)
    rec = np.array([(r.level, r.r) for r in f.records])
    R = np.array([(r.level, r.n, r.r, r.w) for r in f.records], dtype=float)
    for k in range(depth, 1, -1):
        q = R[R[:, 0] == k]
        m = q[:, 1] + q[:, 2]
        print(f"   level {k}: pivots {len(q)} m mean {m.mean():.0f} max {m.max():.0f}  w mean {q[:, 3].mean():.0f} max "
              f"{q[:, 3].max():.0f}  getrf {(2 / 3 * m ** 3).sum() / 1e9:.1f} GF  X {(2 * m * m * q[:, 3]).sum() / 1e9:.1f} GF"
              f"  Schur(full) {(2 * q[:, 1] * q[:, 3] ** 2).sum() / 1e9:.1f} GF")
    print(f"== {name}: factorize {t1 - t0:.2f}s residual {res:.3e} (ref Morton {float(g['resid_morton']):.3e} "
          f"colour9 {float(g['resid_colour9']):.3e}) r_m {f.r_m} top {f.top_dim} (ref {int(g['top_colour9'])})")
    xc, xm = g["x_colour9"], g["x_morton"]
    rel = lambda a, c: np.linalg.norm(a - c) / np.linalg.norm(c)
    print(f"   x vs colour9 {rel(x, xc):.3e}  vs Morton {rel(x, xm):.3e}  ref Morton vs colour9 {rel(xm, xc):.3e}")
    rs = dict(map(tuple, g["rank_sum_colour9"])) if "rank_sum_colour9" in g else {}
    mc = dict(map(tuple, g["max_cond_colour9"])) if "max_cond_colour9" in g else {}
    st = {int(r[0]): r for r in g["stats_colour9"]}
    for k in range(depth, 1, -1):
        s = f.level_stats[k]
        rsum = int(rec[rec[:, 0] == k, 1].sum())
        print(f"   level {k}: rank sum {rsum:7d} (ref {int(rs.get(k, -1)):7d})  max cond {f.max_cond[k]:.2e} "
              f"(ref {mc.get(k, float('nan')):.2e})  fills {s.fillins_compressed:6d} (ref {int(st[k][3]):6d})  "
              f"max rank {s.max_rank} (ref {int(st[k][2])})")
    print(f"   pivots over 1e12: {len(f.singular_pivots)} {f.singular_pivots[:6]}", flush=True)
    del f, store
