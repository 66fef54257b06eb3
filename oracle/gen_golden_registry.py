"""Generate tests/golden/registry_*.npz from the REAL reference package (build container only):
IfmmSolver(kernel=K, a=1e-3, tol=1e-10, p=6) on 4,000 seeded points in [-1, 1]^2 for every
kernel of the reference registry (ifmm/kernels.py:160-170), plus the inverse-quadric kernel in
exact mode (tol = 0) on 1,024 points.  Stores b, the reference solution, residual and r_m;
a kernel whose reference run raises stores the exception instead.

Usage:  OMP_NUM_THREADS=1 OPENBLAS_NUM_THREADS=1 python oracle/gen_golden_registry.py [KERNEL ...]
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(HERE))
import ifmm  # noqa: E402

OUT = os.path.join(os.path.dirname(HERE), "tests", "golden", "registry_{}.npz")
KERNELS = ["log", "laplace3d", "biharmonic", "bessel-y0", "inverse-quadric", "inverse-multiquadric", "helmholtz3d",
           "gaussian", "multiquadric"]


def run(name, kernel, n, tol, p):
    rng = np.random.default_rng(0)
    X = 2.0 * rng.random((n, 2)) - 1.0
    b = rng.standard_normal(n)
    t0 = time.perf_counter()
    try:
        est = ifmm.IfmmSolver(kernel=kernel, a=1e-3, tol=tol, p=p).fit(X)
        x = est.solve(b)
        res = np.linalg.norm(est.matvec(x) - b) / np.linalg.norm(b)
        # the same system eliminated in the GPU's colour order by the CPU oracle (a
        # restatement pinned bit-exactly to the reference in Morton order)
        from oracle import ifmm_oracle as O
        spec = O.KernelSpec(kernel, a=1e-3)
        T = O.build_tree(X, est.tree_.depth)
        fo = O.factorize(O.init_operators(T, spec, p, tol), order="colour9", on_singular="record")
        xo = O.solve(fo, b)
        res9 = np.linalg.norm(O.fmm_matvec(O.init_operators(T, spec, p, tol), xo) - b) / np.linalg.norm(b)
        np.savez_compressed(OUT.format(name), n=n, kernel=kernel, tol=tol, p=p, depth=est.tree_.depth, b=b, x=x,
                            resid=res, resid_colour9=res9, x_colour9=xo, r_m=est.factorization_.r_m, error="")
        print(f"{name}: residual {res:.2e} (colour order {res9:.2e}) r_m {est.factorization_.r_m} depth "
              f"{est.tree_.depth} ({time.perf_counter() - t0:.1f} s)", flush=True)
    except Exception as e:  # the reference's own failure is the expected behaviour
        np.savez_compressed(OUT.format(name), n=n, kernel=kernel, tol=tol, p=p, b=b, error=f"{type(e).__name__}: {e}")
        print(f"{name}: {type(e).__name__}: {e} ({time.perf_counter() - t0:.1f} s)", flush=True)


if __name__ == "__main__":
    for k in sys.argv[1:] or KERNELS:
        run(k.replace("-", "_"), k, 4000, 1e-10, 6)
    if not sys.argv[1:]:
        run("exact_inverse_quadric", "inverse-quadric", 1024, 0.0, 6)
