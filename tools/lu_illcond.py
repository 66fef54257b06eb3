"""Ill-conditioned pivot blocks through the batched LU hooks: condition estimate vs
LAPACK dgecon and the backward error of X = S^-1 C vs scipy lu_solve."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
from scipy.linalg import lu_factor, lu_solve  # noqa: E402
from scipy.linalg.lapack import dgecon  # noqa: E402

from paper_1407_1572_b200 import _lib as L  # noqa: E402
from test_gpu_kernels import _run_lu  # noqa: E402


def saddle(rng, n, r, cond):
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    P = Q @ np.diag(np.logspace(0, -np.log10(cond), n)) @ Q.T
    U, _ = np.linalg.qr(rng.standard_normal((n, r)))
    S = np.zeros((n + r, n + r))
    S[:n, :n] = P
    S[:n, n:] = U
    S[n:, :n] = U.T
    return S


rng = np.random.default_rng(1)
for n, r in [(64, 50), (300, 120), (500, 200)]:
    for cond in [1e6, 1e10, 1e12, 1e14]:
        S = saddle(rng, n, r, cond)
        res, info, est = _run_lu(L, [S])
        LU, perm = res[0]
        lu = lu_factor(S)
        rc = dgecon(lu[0], np.linalg.norm(S, 1), norm="1")[0]
        ref = 1.0 / (rc * np.linalg.norm(S, 1))
        wl = 3 * n
        C = np.asfortranarray(rng.standard_normal((n, wl)))
        xt = np.zeros((n, wl + r), order="F")
        xb = np.zeros((r, wl + r), order="F")
        L.check(L.lib.ifmm_test_lu_solve_x(L.ptr(np.asfortranarray(LU)), L.ptr(perm.astype(np.int32)), n, r,
                                           L.ptr(C), wl, L.ptr(xt), L.ptr(xb)))
        Cf = np.zeros((n + r, wl + r))
        Cf[:n, :wl] = C
        Cf[n:, wl:] = -np.eye(r)
        X = np.vstack([xt, xb])
        Xr = lu_solve(lu, Cf)
        be = np.linalg.norm(S @ X - Cf) / (np.linalg.norm(S) * np.linalg.norm(X))
        be_r = np.linalg.norm(S @ Xr - Cf) / (np.linalg.norm(S) * np.linalg.norm(Xr))
        print(f"n={n} r={r} cond~{cond:.0e}: est ||S^-1|| gpu {est[0]:.3e} dgecon {ref:.3e} ratio {est[0] / ref:.3f} "
              f"| X backward err gpu {be:.1e} scipy {be_r:.1e}  diff {np.linalg.norm(X - Xr) / np.linalg.norm(Xr):.1e}",
              flush=True)
