"""Probe (CPU): oracle with explicit inverses instead of LU -> r_m / top-dim sensitivity."""
import sys, numpy as np
import os; _R = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, _R); sys.path.insert(0, os.path.join(_R, 'tests'))
from oracle import ifmm_oracle as O
from conftest import load_golden, golden_kernel
name = sys.argv[1]
g = load_golden(name)
N, depth, p, tol = int(g["N"]), int(g["depth"]), int(g["p"]), float(g["tol"])
pts = O.baseline_points(N, 0); T = O.build_tree(pts, depth)
O.lu_factor = lambda S: (np.linalg.inv(S), None)
O.lu_solve = lambda lu, C: lu[0] @ C
import scipy.linalg.lapack as lp
O.dgecon = lambda a, anorm, norm="1": (1.0 / (anorm * np.linalg.norm(a, 1)), 0)
st = O.init_operators(T, golden_kernel(g), p, tol)
f = O.factorize(st, order="colour9")
x = O.solve(f, g["b"])
st2 = O.init_operators(T, golden_kernel(g), p, tol)
print(name, "inverse-based oracle: r_m", f.r_m, "top", f.top_off[-1], "ranks", [f.st.r(depth, i) for i in range(min(16, 1 << 2*depth))][:16],
      "resid", np.linalg.norm(O.fmm_matvec(st2, x) - g["b"]) / np.linalg.norm(g["b"]), "ref r_m/top", int(g["rm_colour9"]), int(g["top_colour9"]))
