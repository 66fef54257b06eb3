"""Per-level work of the C3 factorization (pivots, m, w, X-solve / LU / Schur
flops) next to the instrumented phase times: achieved TF/s per level and phase.
    python tools/level_work.py [N depth]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1407_1572_b200 as ifmm  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
depth = int(sys.argv[2]) if len(sys.argv) > 2 else 7
rng = np.random.default_rng(0)
pts = 2.0 * rng.random((N, 2)) - 1.0  # bench.py: [0,1]^2 mapped to the reference box
tree = ifmm.build_tree(ifmm.PointSet(2, pts), depth)
kern = ifmm.baseline_kernel("inv_r", N)
store = ifmm.init_operators(tree, kern, p=4, tol=1e-6)
f = ifmm.factorize(store, tree, on_singular="record")  # warm-up
f = ifmm.factorize(store, tree, on_singular="record", timing=True)
R = np.array([(r.level, r.n, r.r, r.w) for r in f.records], dtype=float)
ph = {str(k): v for k, v in f.phase_times_by_level.items()}
for k in range(depth, 1, -1):
    q = R[R[:, 0] == k]
    m = q[:, 1] + q[:, 2]
    xs = (2 * m * m * q[:, 3]).sum()
    lu = (2 / 3 * m ** 3).sum()
    line = (f"level {k}: pivots {len(q):6d} m mean {m.mean():6.0f} max {m.max():5.0f} w mean {q[:, 3].mean():6.0f} "
            f"max {q[:, 3].max():6.0f}  X {xs / 1e9:7.1f} GF  LU {lu / 1e9:6.1f} GF")
    if ph is not None and str(k) in ph:
        p = ph[str(k)]
        line += f"  | x_solve {p['x_solve']:6.1f} ms = {xs / p['x_solve'] / 1e9:5.1f} TF/s  lu {p['lu']:5.1f} ms"
    print(line, flush=True)
