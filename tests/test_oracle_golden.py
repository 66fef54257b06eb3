"""Pin the CPU oracle against outputs of the real reference (tests/golden, made by
oracle/gen_golden.py).  Tree/lists must be bit-exact; operators and solutions match
to rounding (the restatement reproduces the reference's arithmetic order)."""
import numpy as np
import pytest

from conftest import golden_kernel, load_golden
from oracle import ifmm_oracle as O

CASES = ["c1_invr", "log_2k", "exact_512", "reglog_1k", "d4_invr"]


def _setup(name):
    g = load_golden(name)
    N, depth = int(g["N"]), int(g["depth"])
    pts = O.baseline_points(N, seed=0)
    return g, pts, O.build_tree(pts, depth), golden_kernel(g)


@pytest.mark.parametrize("name", CASES + ["c2_log"])  # C2 itself: tree/lists only (its oracle run takes minutes)
def test_tree_lists_bit_exact(name):
    g, pts, T, _ = _setup(name)
    assert np.array_equal(T.perm, g["perm"])
    assert np.array_equal(T.leaf_off, g["leaf_off"])
    for k in range(1, int(g["depth"]) + 1):
        for i in range(T.n_clusters(k)):
            nb = g[f"nbr{k}"][i]
            il = g[f"il{k}"][i]
            assert T.nbr[k][i] == list(nb[nb >= 0])
            assert T.ilist[k][i] == list(il[il >= 0])


@pytest.mark.parametrize("name", CASES)
def test_init_and_matvec(name):
    g, pts, T, spec = _setup(name)
    st = O.init_operators(T, spec, int(g["p"]), float(g["tol"]))
    for k in range(2, int(g["depth"]) + 1):
        assert np.array_equal([st.r(k, i) for i in range(T.n_clusters(k))], g[f"rank0_{k}"])
    mv = O.fmm_matvec(st, g["xm"])
    assert np.linalg.norm(mv - g["mv"]) <= 1e-13 * np.linalg.norm(g["mv"])


@pytest.mark.parametrize("name", ["c1_invr", "log_2k", "exact_512", "reglog_1k"])
@pytest.mark.parametrize("order", ["morton", "colour9"])
def test_factor_solve_matches_reference(name, order):
    g, pts, T, spec = _setup(name)
    st = O.init_operators(T, spec, int(g["p"]), float(g["tol"]))
    fac = O.factorize(st, order=order)
    x = O.solve(fac, g["b"])
    ref = g[f"x_{order}"]
    # the oracle repeats the reference's arithmetic operation for operation (same numpy /
    # LAPACK calls in the same order, one BLAS thread): bit-identical solutions
    assert np.array_equal(x, ref), np.linalg.norm(x - ref) / np.linalg.norm(ref)
    assert fac.r_m == int(g[f"rm_{order}"])
    assert int(fac.top_off[-1]) == int(g[f"top_{order}"])


def test_exact_mode_matches_dense_lu():
    g, pts, T, spec = _setup("exact_512")
    st = O.init_operators(T, spec, int(g["p"]), 0.0)
    x = O.solve(O.factorize(st, order="colour9"), g["phi"])
    assert np.linalg.norm(x - g["x_dense"]) <= 1e-11 * np.linalg.norm(g["x_dense"])


def test_nrhs_solve_equals_columnwise():
    g, pts, T, spec = _setup("log_2k")
    st = O.init_operators(T, spec, int(g["p"]), float(g["tol"]))
    fac = O.factorize(st, order="colour9")
    B = np.stack([g["b"], g["xm"]], axis=1)
    X = O.solve(fac, B)
    for c, v in enumerate((g["b"], g["xm"])):
        ref = O.solve(fac, v)
        assert np.linalg.norm(X[:, c] - ref) <= 1e-13 * np.linalg.norm(ref)


def test_oracle_rank_control_extension():
    """oracle/_consolidate (the checker of the GPU's rank_tol extension, not reference
    behaviour): ranks shrink, the residual against the compressed operator stays
    near the truncation tolerance, in both elimination orders; off by default."""
    from oracle import ifmm_oracle as O
    N, depth, p, tol = 1024, 2, 4, 1e-6
    pts = O.baseline_points(N, seed=0)
    spec = O.baseline_kernel("log_r", N)
    tree = O.build_tree(pts, depth)
    b = O.baseline_rhs(N, "normal")
    f0 = O.factorize(O.init_operators(tree, spec, p, tol), order="colour9")
    assert f0.rank_control == [0, 0]
    for order in ("colour9", "morton"):
        f1 = O.factorize(O.init_operators(tree, spec, p, tol), order=order, rank_tol=1e-7)
        assert 0 < f1.rank_control[1] < f1.rank_control[0]
        assert f1.top_off[-1] < f0.top_off[-1]
        x = O.solve(f1, b)
        res = np.linalg.norm(O.fmm_matvec(O.init_operators(tree, spec, p, tol), x) - b) / np.linalg.norm(b)
        assert res <= 10 * tol, (order, res)


def test_oracle_sparse_tree_extension():
    """oracle build_tree(allow_empty=True) (the checker of the GPU's allow_empty_leaves
    extension, not reference behaviour): exact mode equals the dense LU solution on a tree
    with empty cells; with compression no fill is kept dense; the default still raises."""
    import bench
    from oracle import ifmm_oracle as O
    n, depth = 1024, 3
    X = bench.mixture_points(n)
    with pytest.raises(ValueError, match="empty"):
        O.build_tree(X, depth)
    T = O.build_tree(X, depth, allow_empty=True)
    assert (np.diff(T.leaf_off) == 0).any()
    spec = O.baseline_kernel("inv_r", n)
    b = np.random.default_rng(1).standard_normal(n)
    x = O.solve(O.factorize(O.init_operators(T, spec, 4, 0.0)), b)
    xd = np.linalg.solve(O.dense_matrix(spec, X), b)
    assert np.linalg.norm(x - xd) / np.linalg.norm(xd) <= 1e-10
    fac = O.factorize(O.init_operators(T, spec, 4, 1e-6), order="colour9")
    assert sum(s.dense_kept for s in fac.stats.values()) == 0
    x = O.solve(fac, b)
    res = np.linalg.norm(O.fmm_matvec(O.init_operators(T, spec, 4, 1e-6), x) - b) / np.linalg.norm(b)
    assert res <= 1e-4
