"""Probe (CPU): per-level pivot condition numbers of the reference algorithm (oracle, LU) -- DESIGN.md 5.
   usage: python tools/oracle_pivot_cond.py N depth {morton|colour9}"""
import sys, numpy as np, time
import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from threadpoolctl import threadpool_limits
threadpool_limits(1)
from oracle import ifmm_oracle as O
from scipy.linalg.lapack import dgecon
N, depth = int(sys.argv[1]), int(sys.argv[2]); order = sys.argv[3]
pts = O.baseline_points(N, 0); spec = O.baseline_kernel("inv_r", N)
T = O.build_tree(pts, depth); st = O.init_operators(T, spec, 4, 1e-6)
conds = {}
orig = O._eliminate
def el(st, k, i, tol, fac, stats, ils, dead):
    orig(st, k, i, tol, fac, stats, ils, dead)
    lu = fac.recs[-1].lu
    U = st.U[(k, i)]
    # exact 1-norm cond of the pivot from its LU (small m)
    m = lu[0].shape[0]
    from scipy.linalg import lu_solve
    inv = lu_solve(lu, np.eye(m))
    L = np.tril(lu[0], -1) + np.eye(m); Uu = np.triu(lu[0])
    A = L @ Uu
    piv = lu[1]; Pm = np.eye(m)
    for a, b in enumerate(piv): Pm[[a, b]] = Pm[[b, a]]
    S = Pm.T @ A
    c = np.linalg.norm(S, 1) * np.linalg.norm(inv, 1)
    conds.setdefault(k, []).append(c)
O._eliminate = el
t0 = time.time()
fac = O.factorize(st, order=order)
b = O.baseline_rhs(N, "normal"); x = O.solve(fac, b)
st2 = O.init_operators(T, spec, 4, 1e-6)
print(order, "time", time.time()-t0, "resid", np.linalg.norm(O.fmm_matvec(st2, x) - b)/np.linalg.norm(b))
for k in sorted(conds, reverse=True):
    c = np.array(conds[k]); print(f"level {k}: max cond {c.max():.3e} geo-mean {np.exp(np.log(c).mean()):.3e}")
