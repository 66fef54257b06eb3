"""Generate tests/golden/*.npz from the REAL reference package (build container only).

Usage:  OMP_NUM_THREADS=1 OPENBLAS_NUM_THREADS=1 python oracle/gen_golden.py

The reference (`/root/reference/pkg/src/ifmm`) is imported read-only.  Two
elimination orders are recorded:
  * "morton": the reference's own `factorize` (ifmm/solver.py:106-153);
  * "colour9": the same private functions (`_form_parent_p2p`,
    `_release_level_m2l`, `_eliminate_cluster`, `_factor_top_level`,
    ifmm/solver.py:156-546) driven in the colour-major order the GPU uses.
Fixtures hold seeds + outputs only (no reference source).
"""
import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")

import ifmm  # noqa: E402
from ifmm import solver as rsolver  # noqa: E402
from ifmm.kernels import Kernel  # noqa: E402

from oracle import ifmm_oracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")

CASES = {
    # name: (N, kernel, a, depth, p, tol)
    "c1_invr": (4096, "inv_r", 0.001, 3, 4, 1e-8),
    "log_2k": (2048, "log_r", 0.001, 3, 5, 1e-6),
    "exact_512": (512, "inv_r", 0.001, 2, 4, 0.0),
    "reglog_1k": (1024, "log", 0.001, 2, 4, 1e-10),
    "d4_invr": (16384, "inv_r", 0.001, 4, 4, 1e-6),
    # BASELINE C2 itself (N = 65,536, log|x-y|, depth 5, p = 5, eps = 1e-6)
    "c2_log": (65536, "log_r", 0.001, 5, 5, 1e-6),
    # C3's parameters one level shallower (N = 262,144, depth 6): the largest case the reference
    # finishes in minutes (C3 itself needs ~1 h and ~70 GB)
    "c3_262k": (262144, "inv_r", 0.001, 6, 4, 1e-6),
}


def ref_kernel(name, a, n):
    if name in ("inv_r", "log_r"):
        spec = O.baseline_kernel(name, n)
        return spec, Kernel(name, a, lambda r: O.kernel_eval(spec, np.asarray(r, dtype=float)))
    return O.KernelSpec(name, a=a), ifmm.make_kernel(name, a=a)


def colour9_factorize(store, tree, tol):
    """Reference private functions driven in colour-major order."""
    for lv in tree.levels.values():
        for c in lv:
            c.eliminated = False
    fact = rsolver.IfmmFactorization(store=store, tree=tree, tol=tol)
    fact.r_m = store.max_init_rank
    kappa = tree.depth
    ot = O.Tree(kappa, tree.dim, None, None, None,
                {k: np.array([c.grid for c in tree.levels[k]]) for k in tree.levels}, None, None)
    for k in range(kappa, 1, -1):
        if k < kappa:
            rsolver._form_parent_p2p(store, tree, k)
            rsolver._release_level_m2l(store, k + 1)
        stats = rsolver.LevelStats(clusters=len(tree.levels[k]))
        fact.level_stats[k] = stats
        ilists = [set(c.interaction_list) for c in tree.levels[k]]
        for batch in O.elimination_order(ot, k, "colour9"):
            for i in batch:
                rsolver._eliminate_cluster(store, tree, k, int(i), tol, fact, stats, ilists)
        fact.r_m = max(fact.r_m, stats.max_rank)
    rsolver._factor_top_level(fact)
    rsolver._release_level_m2l(store, 2)
    return fact


def pack_lists(tree):
    out = {}
    for k in range(1, tree.depth + 1):
        nc = len(tree.levels[k])
        nb = -np.ones((nc, 9), dtype=np.int32)
        il = -np.ones((nc, 27), dtype=np.int32)
        for c in tree.levels[k]:
            nb[c.index, :len(c.neighbors)] = c.neighbors
            il[c.index, :len(c.interaction_list)] = c.interaction_list
        out[f"nbr{k}"] = nb
        out[f"il{k}"] = il
    return out


def run_case(name, N, kern, a, depth, p, tol):
    pts = O.baseline_points(N, seed=0)
    spec, K = ref_kernel(kern, a, N)
    ps = ifmm.PointSet(2, pts)
    tree = ifmm.compute_lists(ifmm.build_tree(ps, depth))
    rng = np.random.default_rng(11)
    xm = rng.standard_normal(N)
    sigma = rng.uniform(-1.0, 1.0, N)
    b = O.baseline_rhs(N, "normal")
    res = dict(N=N, depth=depth, p=p, tol=tol, a=a, kernel=kern, scale=spec.scale, shift=spec.shift,
               perm=tree.point_permutation.astype(np.int64),
               leaf_off=np.array([c.point_range[0] for c in tree.levels[depth]] + [N], dtype=np.int64),
               xm=xm, b=b, sigma=sigma)
    res.update(pack_lists(tree))
    st = ifmm.init_operators(tree, K, p=p, tol=tol)
    res["mv"] = ifmm.fmm_matvec(st, tree, xm)
    for k in range(2, depth + 1):
        res[f"rank0_{k}"] = np.array([st.rank(k, c.index) for c in tree.levels[k]], dtype=np.int32)
    # the level-2 far operator U_i M2L_ij U_j^T is basis-invariant: keep one block
    if tol > 0:
        i, j = 0, tree.levels[2][0].interaction_list[0]
        res["far_2_0_j"] = np.array([j])
        res["far_2_0"] = st.l2p[(2, i)] @ st.m2l[(2, i, j)] @ st.l2p[(2, j)].T
    t0 = time.time()
    fm = ifmm.factorize(st, tree, tol=tol)
    tfm = time.time() - t0
    res["x_morton"] = ifmm.solve(fm, b)
    res["rm_morton"] = fm.r_m
    res["top_morton"] = int(fm.top_offsets[-1])
    res["stats_morton"] = np.array([[k, s.clusters, s.max_rank, s.fillins_compressed, s.fillins_dense_kept]
                                    for k, s in sorted(fm.level_stats.items())], dtype=np.int64)
    st2 = ifmm.init_operators(tree, K, p=p, tol=tol)
    fc = colour9_factorize(st2, tree, tol)
    res["x_colour9"] = ifmm.solve(fc, b)
    res["rm_colour9"] = fc.r_m
    res["top_colour9"] = int(fc.top_offsets[-1])
    res["stats_colour9"] = np.array([[k, s.clusters, s.max_rank, s.fillins_compressed, s.fillins_dense_kept]
                                     for k, s in sorted(fc.level_stats.items())], dtype=np.int64)
    st3 = ifmm.init_operators(tree, K, p=p, tol=tol)
    res["resid_morton"] = np.linalg.norm(ifmm.fmm_matvec(st3, tree, res["x_morton"]) - b) / np.linalg.norm(b)
    res["resid_colour9"] = np.linalg.norm(ifmm.fmm_matvec(st3, tree, res["x_colour9"]) - b) / np.linalg.norm(b)
    if N <= 4096:
        A = ifmm.assemble_dense(K, ps) if kern not in ("inv_r", "log_r") else O.dense_matrix(spec, pts)
        phi = A @ sigma
        res["phi"] = phi
        res["x_dense"] = np.linalg.solve(A, phi)
        res["x_ifmm_phi"] = ifmm.solve(fm, phi)
    print(f"{name}: t_f(morton)={tfm:.2f}s r_m={fm.r_m}/{fc.r_m} top={res['top_morton']}/{res['top_colour9']} "
          f"resid={res['resid_morton']:.2e}/{res['resid_colour9']:.2e}")
    return res


def main():
    os.makedirs(OUT, exist_ok=True)
    only = sys.argv[1:]
    for name, cfg in CASES.items():
        if only and name not in only:
            continue
        res = run_case(name, *cfg)
        if cfg[0] > 100000:  # keep the large fixture small: what its tests read
            for k in ("sigma", "xm", "mv"):
                res.pop(k, None)
            res["perm"] = res["perm"].astype(np.int32)
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **res)


if __name__ == "__main__":
    main()
