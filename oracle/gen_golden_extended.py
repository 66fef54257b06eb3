"""Generate tests/golden/extended_256.npz from the REAL reference (build container only):
the extended sparse system of ifmm/operators.py:333-486 on a small store.

Usage:  OMP_NUM_THREADS=1 OPENBLAS_NUM_THREADS=1 python oracle/gen_golden_extended.py

Stored: the slot layout (extended_layout), the leaf particle-equation rows of
leaf 0 (kernel values: basis-independent), the number of nonzeros, and the
original-unknown part of the extended solve for a seeded rhs (independent of
the sign / rotation freedom of the SVD bases).  Fixtures hold outputs only.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")

import ifmm  # noqa: E402
from ifmm import operators as rops  # noqa: E402

from oracle import ifmm_oracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(HERE), "tests", "golden", "extended_256.npz")
SYM = {"x": 0, "y": 1, "z": 2}


def main():
    N, depth, p, tol, a = 256, 2, 4, 1e-10, 0.001
    pts = O.baseline_points(N, seed=0)
    tree = ifmm.compute_lists(ifmm.build_tree(ifmm.PointSet(2, pts), depth))
    st = ifmm.init_operators(tree, ifmm.make_kernel("log", a=a), p=p, tol=tol)
    A, slots = rops.assemble_extended_dense(st, tree)
    b = np.random.default_rng(5).standard_normal(N)
    xe = np.linalg.solve(A, rops.extended_rhs(st, tree, b))
    x = rops.extended_restrict_x(st, tree, xe)
    n0 = slots[0][3]
    np.savez_compressed(
        OUT, N=N, depth=depth, p=p, tol=tol, a=a,
        slots=np.array([[SYM[s], k, i, d] for s, k, i, d in slots], dtype=np.int32),
        leaf0_rows=A[:n0, :], nnz=np.count_nonzero(A), b=b, x=x,
        resid=np.linalg.norm(ifmm.fmm_matvec(st, tree, x) - b) / np.linalg.norm(b))
    print(f"extended_256: dim {A.shape[0]}, nnz {np.count_nonzero(A)}")


if __name__ == "__main__":
    main()
