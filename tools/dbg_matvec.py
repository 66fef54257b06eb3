"""Debug: GPU fmm_matvec vs the oracle's and the dense product for one kernel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1407_1572_b200 as ifmm  # noqa: E402
from oracle import ifmm_oracle as O  # noqa: E402

kern, n, depth, p, tol = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), float(sys.argv[5])
a = float(sys.argv[6]) if len(sys.argv) > 6 else 1e-3
rng = np.random.default_rng(0)
X = 2.0 * rng.random((n, 2)) - 1.0
x = rng.standard_normal(n)
tree = ifmm.build_tree(ifmm.PointSet(2, X), depth)
store = ifmm.init_operators(tree, ifmm.make_kernel(kern, a=a), p=p, tol=tol)
yg = ifmm.fmm_matvec(store, tree, x)
T = O.build_tree(X, depth)
spec = O.KernelSpec(kern, a=a)
st = O.init_operators(T, spec, p, tol)
yo = O.fmm_matvec(st, x)
A = O.dense_matrix(spec, X)
yd = A @ x
print(f"{kern} a={a} tol={tol}: |gpu-oracle|/|oracle| {np.linalg.norm(yg - yo) / np.linalg.norm(yo):.3e}  "
      f"|gpu-dense| {np.linalg.norm(yg - yd) / np.linalg.norm(yd):.3e}  |oracle-dense| {np.linalg.norm(yo - yd) / np.linalg.norm(yd):.3e}")
# near field only: leaf P2P blocks vs the kernel
k = depth
errs = []
for i in range(1 << (2 * k)):
    for j in tree.levels[k][i].neighbors:
        Bg = store.p2p[(k, i, j)]
        pi = T.points[T.leaf_off[i]:T.leaf_off[i + 1]]
        pj = T.points[T.leaf_off[j]:T.leaf_off[j + 1]]
        Bo = O.kblock(spec, pi, pj)
        if i == j:
            Bo = Bo + np.eye(len(pi))
        errs.append(np.abs(Bg - Bo).max() / max(np.abs(Bo).max(), 1e-300))
print("max rel error of leaf P2P blocks vs kernel:", max(errs))
