"""Per-phase / per-level device times of one factorization of a bench config.

    python tools/phase_times.py [CONFIG] [REPS]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_1407_1572_b200 as ifmm  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
N, kern, depth, p, tol, nrhs = bench.CONFIGS[name]
pts = 2.0 * np.random.default_rng(0).random((N, 2)) - 1.0
b = np.random.default_rng([0, 1]).standard_normal(N)
tree = ifmm.build_tree(ifmm.PointSet(2, pts), depth)
store = ifmm.init_operators(tree, ifmm.baseline_kernel(kern, N), p=p, tol=tol)
fact = None
for r in range(reps):
    fact = None  # free the previous factorization first (as bench.py does): its slabs return to the cache
    t0 = time.perf_counter()
    fact = ifmm.factorize(store, tree, pivot_condition_limit=1e15, timing=(r == reps - 1))
    t1 = time.perf_counter()
    print(f"rep {r}: factorize wall {1e3 * (t1 - t0):.1f} ms (lib {fact.factor_ms:.1f} ms)", flush=True)
x = ifmm.solve(fact, b)
res = np.linalg.norm(ifmm.fmm_matvec(store, tree, x) - b) / np.linalg.norm(b)
import hashlib  # noqa: E402
print(f"{name}: residual {res:.3e} r_m {fact.r_m} top {fact.top_dim} x {hashlib.md5(x.tobytes()).hexdigest()[:12]}")
print("phases:", {k: round(v[0], 1) for k, v in fact.phase_times.items()})
for k, d in sorted(fact.phase_times_by_level.items(), reverse=True):
    print(f"  level {k}: " + " ".join(f"{p}={v:.1f}" for p, v in d.items() if v))
w = fact.work
ph = fact.phase_times
print(f"schur {w['flops_schur'] / 1e12:.3f} TF in {ph['schur_gemm'][0]:.1f} ms = "
      f"{w['flops_schur'] / ph['schur_gemm'][0] / 1e9:.1f} TF/s")
