"""Clustered inputs on a uniform tree whose empty cells are accepted
(build_tree(..., allow_empty_leaves=True); SURVEY.md 8f item 2 asks for an
adaptive tree -- this is the uniform-tree step toward BASELINE config 4, whose
Gaussian-mixture input it runs).  The reference raises on an empty leaf
(ifmm/geometry.py:191-195), so there is no reference output: the checks are the
dense LU of the true kernel matrix in exact mode, the residual against the
compressed operator, and agreement between the parity path and rank control.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ifmm():
    import paper_1407_1572_b200 as m
    from paper_1407_1572_b200 import _lib
    if _lib.lib.ifmm_device_count() == 0:
        pytest.skip("no CUDA device")
    return m


def _mixture(n):
    import bench
    return bench.mixture_points(n)


def test_empty_leaf_still_raises_by_default(ifmm):
    X = _mixture(4096)
    with pytest.raises(ValueError, match="empty"):
        ifmm.build_tree(ifmm.PointSet(2, X), 4)
    tree = ifmm.build_tree(ifmm.PointSet(2, X), 4, allow_empty_leaves=True)
    cnt = np.diff(tree.leaf_offsets)
    assert (cnt == 0).sum() > 50 and cnt.sum() == 4096


def test_exact_mode_matches_dense_lu_with_empty_cells(ifmm):
    """tol = 0 (identity bases, no compression): the elimination over a tree with
    empty cells reproduces the dense LU solution of the true kernel matrix."""
    from oracle import ifmm_oracle as O
    n, depth = 2048, 3
    X = _mixture(n)
    kern = ifmm.baseline_kernel("inv_r", n)
    tree = ifmm.build_tree(ifmm.PointSet(2, X), depth, allow_empty_leaves=True)
    assert (np.diff(tree.leaf_offsets) == 0).any()
    store = ifmm.init_operators(tree, kern, p=4, tol=0.0)
    b = np.random.default_rng(1).standard_normal(n)
    x = ifmm.solve(ifmm.factorize(store, tree), b)
    A = O.dense_matrix(O.baseline_kernel("inv_r", n), X)
    xd = np.linalg.solve(A, b)
    assert np.linalg.norm(x - xd) / np.linalg.norm(xd) <= 1e-10


@pytest.mark.parametrize("n,depth,p,tol,rank_tol,bound", [
    (4096, 4, 4, 1e-6, None, 1e-4),
    (65536, 6, 4, 1e-6, None, 1e-3),     # failed before full-rank fills were absorbed (residual 4.8, 76 s)
    (65536, 6, 4, 1e-6, 1e-7, 1e-3),
    (65536, 6, 6, 1e-10, 1e-9, 1e-5),
])
def test_mixture_on_a_tree_with_empty_cells(ifmm, n, depth, p, tol, rank_tol, bound):
    X = _mixture(n)
    kern = ifmm.baseline_kernel("inv_r", n)
    tree = ifmm.build_tree(ifmm.PointSet(2, X), depth, allow_empty_leaves=True)
    store = ifmm.init_operators(tree, kern, p=p, tol=tol)
    f = ifmm.factorize(store, tree, on_singular="record", rank_tol=rank_tol)
    # no dense coupling chains through the sparse regions: every well-separated fill is absorbed
    assert sum(f.level_stats[k].fillins_dense_kept for k in range(2, depth + 1)) == 0
    assert f.factor_ms < 5000
    b = np.random.default_rng(1).standard_normal(n)
    nb = np.linalg.norm(b)
    x = ifmm.solve(f, b)
    res = np.linalg.norm(ifmm.fmm_matvec(store, tree, x) - b) / nb
    assert res <= bound, res
    x2 = ifmm.solve(f, b, refine=2)
    res2 = np.linalg.norm(ifmm.fmm_matvec(store, tree, x2) - b) / nb
    assert res2 <= max(1e-3 * bound, 100 * tol), (res, res2)


def test_sparse_tree_through_the_estimator_and_sharded(ifmm):
    """IfmmSolver(allow_empty_leaves=True, rank_tol=...) on the mixture, and the same
    factorization on 4 virtual ranks (bit-identical to one GPU)."""
    from paper_1407_1572_b200 import distributed as D
    n = 16384
    X = _mixture(n)
    k = ifmm.baseline_kernel("inv_r", n)
    est = ifmm.IfmmSolver(kernel="inv_r", tol=1e-6, p=4, depth=5, kernel_scale=k.scale, kernel_shift=k.shift,
                          rank_tol=1e-7, allow_empty_leaves=True).fit(X)
    b = np.random.default_rng(1).standard_normal(n)
    x = est.solve(b)
    assert np.linalg.norm(est.matvec(x) - b) / np.linalg.norm(b) <= 1e-3
    fs = D.factorize_emulated(est.store_, est.tree_, 4, rank_tol=1e-7)
    xs = D.solve_emulated(fs, b)
    assert np.array_equal(xs[0], x) and np.array_equal(xs[3], x)


@pytest.mark.parametrize("rank_tol", [None, 1e-7])
def test_sparse_tree_against_the_oracle(ifmm, rank_tol):
    """The oracle's restatement of the same extension (oracle build_tree(allow_empty=True):
    empty clusters skipped, full-rank fills absorbed), same colour order: tree bit-exact,
    ranks and top dimension within 5 %, residual within 2x, solutions within the
    compression error."""
    from oracle import ifmm_oracle as O
    n, depth, p, tol = 4096, 4, 4, 1e-6
    X = _mixture(n)
    tree = ifmm.build_tree(ifmm.PointSet(2, X), depth, allow_empty_leaves=True)
    T = O.build_tree(X, depth, allow_empty=True)
    assert np.array_equal(tree.point_permutation, T.perm)
    assert np.array_equal(tree.leaf_offsets, T.leaf_off)
    store = ifmm.init_operators(tree, ifmm.baseline_kernel("inv_r", n), p=p, tol=tol)
    f = ifmm.factorize(store, tree, rank_tol=rank_tol)
    b = np.random.default_rng(1).standard_normal(n)
    x = ifmm.solve(f, b)
    res = np.linalg.norm(ifmm.fmm_matvec(store, tree, x) - b) / np.linalg.norm(b)
    spec = O.baseline_kernel("inv_r", n)
    fo = O.factorize(O.init_operators(T, spec, p, tol), order="colour9", rank_tol=rank_tol)
    xo = O.solve(fo, b)
    res_o = np.linalg.norm(O.fmm_matvec(O.init_operators(T, spec, p, tol), xo) - b) / np.linalg.norm(b)
    assert res <= max(10 * tol, 2 * res_o), (res, res_o)
    # empty clusters carry no unknowns: the GPU keeps zero-size records for them, the oracle none
    assert sum(1 for r in f.records if r.n + r.r > 0) == len(fo.recs)
    assert abs(f.top_dim - int(fo.top_off[-1])) <= 0.05 * fo.top_off[-1], (f.top_dim, fo.top_off[-1])
    rec = np.array([(r.level, r.r) for r in f.records])
    for k in range(depth, 1, -1):
        ro = sum(r.r for r in fo.recs if r.level == k)
        assert abs(int(rec[rec[:, 0] == k, 1].sum()) - ro) <= 0.05 * ro, (k, ro)
    assert np.linalg.norm(x - xo) / np.linalg.norm(xo) <= 100 * tol


def test_mixed_size_batches_against_the_oracle_run(ifmm):
    """N = 262,144 on a depth-7 tree: colour batches of ~1,800 pivots that mix few-point and
    ~900-point cells, so the pivots are factored by size class (own pivots reordered).  The
    fill states must follow that order (they did not at first: 37 absorbed fills were booked as
    kept dense and the residual was 2.8e-2).  Against the oracle's run of the same system
    (tests/golden/mixture_262k_rank_control.json, 145 s of one core): records, no dense fill,
    rank sums within 3 %, top dimension within 5 %."""
    import json
    import os
    from conftest import GOLDEN
    g = json.load(open(os.path.join(GOLDEN, "mixture_262k_rank_control.json")))
    n, depth = 262144, 7
    X = _mixture(n)
    tree = ifmm.build_tree(ifmm.PointSet(2, X), depth, allow_empty_leaves=True)
    store = ifmm.init_operators(tree, ifmm.baseline_kernel("inv_r", n), p=4, tol=1e-6)
    f = ifmm.factorize(store, tree, on_singular="record", rank_tol=1e-7)
    assert sum(f.level_stats[k].fillins_dense_kept for k in range(2, depth + 1)) == 0
    recs = f.records
    assert sum(1 for r in recs if r.n + r.r > 0) == g["records"]
    rec = np.array([(r.level, r.r) for r in recs])
    for k in range(depth, 1, -1):
        ro = g["rank_sum"][str(k)]
        assert abs(int(rec[rec[:, 0] == k, 1].sum()) - ro) <= 0.03 * ro, (k, ro)
    assert abs(f.top_dim - g["top_dim"]) <= 0.05 * g["top_dim"]
    b = np.random.default_rng(1).standard_normal(n)
    x = ifmm.solve(f, b)
    res = np.linalg.norm(ifmm.fmm_matvec(store, tree, x) - b) / np.linalg.norm(b)
    assert res <= 5e-3, res  # the oracle: 3.0e-4; the clipped mixture is ill-conditioned (pivots near 1e12)
    x2 = ifmm.solve(f, b, refine=2)
    assert np.linalg.norm(ifmm.fmm_matvec(store, tree, x2) - b) / np.linalg.norm(b) <= 1e-5


def test_mixed_size_batches_sharded(ifmm):
    """The same 262,144-point system on 2 and 4 virtual ranks: the size-class order of each
    rank's own pivots and the per-class panel widths come from the whole batch, so the sharded
    result is bit-identical to one GPU."""
    from paper_1407_1572_b200 import distributed as D
    n, depth = 262144, 7
    X = _mixture(n)
    b = np.random.default_rng(1).standard_normal(n)
    tree = ifmm.build_tree(ifmm.PointSet(2, X), depth, allow_empty_leaves=True)
    store = ifmm.init_operators(tree, ifmm.baseline_kernel("inv_r", n), p=4, tol=1e-6)
    f = ifmm.factorize(store, tree, rank_tol=1e-7, pivot_condition_limit=np.inf)
    x = ifmm.solve(f, b)
    for V in (2, 4):
        fs = D.factorize_emulated(store, tree, V, rank_tol=1e-7, pivot_condition_limit=np.inf)
        xs = D.solve_emulated(fs, b)
        assert np.array_equal(xs[0], x) and np.array_equal(xs[V - 1], x), V
        del fs
