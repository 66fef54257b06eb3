"""Device time of ifmm.solve alone (factorize once, then repeated solves).

    python tools/solve_time.py [CONFIG] [REPS]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1407_1572_b200 as ifmm  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
nq = int(sys.argv[3]) if len(sys.argv) > 3 else 1
N, kern, depth, p, tol, _ = bench.CONFIGS[name]
nrhs = nq
pts = 2.0 * np.random.default_rng(0).random((N, 2)) - 1.0
b = torch.from_numpy(np.random.default_rng([0, 1]).standard_normal((N, nrhs) if nrhs > 1 else N)).cuda()
tree = ifmm.build_tree(ifmm.PointSet(2, pts), depth)
store = ifmm.init_operators(tree, ifmm.baseline_kernel(kern, N), p=p, tol=tol)
fact = ifmm.factorize(store, tree, pivot_condition_limit=1e15)
w = fact.work
for r in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x = ifmm.solve(fact, b)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"solve nrhs={nrhs} {1e3 * dt:.2f} ms  (record bytes {w['solve_bytes'] / 1e9:.1f} GB per rhs; "
          f"{w['solve_bytes'] / dt / 1e9:.0f} GB/s for one pass)")
