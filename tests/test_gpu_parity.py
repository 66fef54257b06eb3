"""GPU parity tests through the public API / C-ABI against the CPU oracle and
the reference goldens (tests/golden, made by oracle/gen_golden.py).

Gates:
  G1 tree / lists / colouring bit-exact;
  G2 exact mode (tol = 0): solution vs dense LU <= 1e-11;
  G3 residual vs the FMM operator <= max(10 eps, 2 x the reference's own
     (Morton-order) residual);
  G4 solution difference vs the reference run in the same (colour9) order:
     <= 10 eps for the log kernel, <= 2 x the reference's own Morton-vs-colour
     difference for 1/r (SURVEY.md finding 5: eps x cond apart);
  G5 initial ranks equal, top-level dimension within 10 %, r_m within 25 %,
     per-level statistics against the reference's.
"""
import numpy as np
import pytest

from conftest import golden_kernel, load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ifmm():
    import paper_1407_1572_b200 as m
    from paper_1407_1572_b200 import _lib
    if _lib.lib.ifmm_device_count() == 0:
        pytest.skip("no CUDA device")
    return m


def _kernel(ifmm, g):
    return ifmm.make_kernel(str(g["kernel"]), a=float(g["a"]), scale=float(g["scale"]), shift=float(g["shift"]))


def _setup(ifmm, name):
    from oracle import ifmm_oracle as O
    g = load_golden(name)
    N, depth = int(g["N"]), int(g["depth"])
    pts = O.baseline_points(N, seed=0)
    tree = ifmm.build_tree(ifmm.PointSet(2, pts), depth)
    return g, pts, tree


CASES = ["c1_invr", "log_2k", "exact_512", "reglog_1k", "d4_invr", "c2_log"]


@pytest.mark.parametrize("name", CASES)
def test_tree_lists_colours_bit_exact(ifmm, name):
    g, pts, tree = _setup(ifmm, name)
    assert np.array_equal(tree.point_permutation, g["perm"])
    assert np.array_equal(tree.leaf_offsets, g["leaf_off"])
    for k in range(1, int(g["depth"]) + 1):
        nbo, nb, ilo, il = tree.lists(k)
        for i in range(1 << (2 * k)):
            ref_nb = g[f"nbr{k}"][i]
            ref_il = g[f"il{k}"][i]
            assert list(nb[nbo[i]:nbo[i + 1]]) == list(ref_nb[ref_nb >= 0])
            assert list(il[ilo[i]:ilo[i + 1]]) == list(ref_il[ref_il >= 0])
        gx, gy = np.arange(1 << k), None
        grid = ifmm.morton_decode(np.arange(1 << (2 * k)), 2, k)
        assert np.array_equal(tree.colours(k), (grid[:, 0] % 3) + 3 * (grid[:, 1] % 3))


@pytest.mark.parametrize("name", CASES)
def test_init_ranks_and_matvec(ifmm, name):
    g, pts, tree = _setup(ifmm, name)
    store = ifmm.init_operators(tree, _kernel(ifmm, g), p=int(g["p"]), tol=float(g["tol"]))
    for k in range(2, int(g["depth"]) + 1):
        assert np.array_equal(store.ranks(k), g[f"rank0_{k}"]), k
    mv = ifmm.fmm_matvec(store, tree, g["xm"])
    assert np.linalg.norm(mv - g["mv"]) <= 1e-12 * np.linalg.norm(g["mv"])
    if "far_2_0" in g and int(g["depth"]) == 2:
        # U M2L U^T is basis-invariant only where the particle axis is physical (leaf level)
        j = int(g["far_2_0_j"][0])
        U0, Uj = store.l2p[(2, 0)], store.l2p[(2, j)]
        far = U0 @ store.m2l[(2, 0, j)] @ Uj.T
        assert np.linalg.norm(far - g["far_2_0"]) <= 1e-12 * np.linalg.norm(g["far_2_0"])


def test_matvec_multi_rhs_equals_columns(ifmm):
    g, pts, tree = _setup(ifmm, "log_2k")
    store = ifmm.init_operators(tree, _kernel(ifmm, g), p=int(g["p"]), tol=float(g["tol"]))
    X = np.stack([g["xm"], g["b"], g["xm"] - g["b"]], axis=1)
    Y = ifmm.fmm_matvec(store, tree, X)
    for c in range(3):
        y = ifmm.fmm_matvec(store, tree, X[:, c])
        assert np.linalg.norm(Y[:, c] - y) <= 1e-14 * np.linalg.norm(y)


@pytest.mark.parametrize("name", ["c1_invr", "log_2k", "reglog_1k", "d4_invr", "c2_log", "c3_262k"])
def test_factor_solve_residual_and_solution(ifmm, name):
    g, pts, tree = _setup(ifmm, name)
    tol = float(g["tol"])
    assert np.array_equal(tree.point_permutation, g["perm"])
    store = ifmm.init_operators(tree, _kernel(ifmm, g), p=int(g["p"]), tol=tol)
    # c3_262k (C3's parameters at N = 262,144) sits at the reference's 1e12
    # pivot-condition limit (at C3 itself the reference exceeds it in both
    # orders, tests/golden/c3_1m.npz): record such pivots instead of raising
    big = name == "c3_262k"
    fact = ifmm.factorize(store, tree, on_singular="record" if big else "raise")
    assert len(fact.singular_pivots) <= (2 if big else 0), fact.singular_pivots
    x = ifmm.solve(fact, g["b"])
    b = g["b"]
    res = np.linalg.norm(ifmm.fmm_matvec(store, tree, x) - b) / np.linalg.norm(b)
    ref_res = float(g["resid_morton"])
    # G3: residual against the compressed operator, vs the reference's own
    assert res <= max(10 * tol, 2 * ref_res), (res, ref_res)
    # G4: solution vs the reference run in the same colour order
    xc = g["x_colour9"]
    diff = np.linalg.norm(x - xc) / np.linalg.norm(xc)
    if str(g["kernel"]).startswith("log"):
        assert diff <= 10 * tol, diff
    else:
        morton_vs_colour = np.linalg.norm(g["x_morton"] - xc) / np.linalg.norm(xc)
        assert diff <= max(10 * tol, 2 * morton_vs_colour), (diff, morton_vs_colour)
    # G5: ranks.  r_m (max ACA rank) is noise-driven near the cutoff: the CPU
    # oracle itself drops from 28 to 16 on reglog_1k when its LU solves are
    # replaced by an explicit inverse, so gate
    # on the top-level dimension (sum of final level-2 ranks) and bound r_m above.
    ref_top = int(g["top_colour9"])
    assert abs(fact.top_dim - ref_top) <= 0.1 * ref_top, (fact.top_dim, ref_top)
    assert fact.r_m <= 1.25 * int(g["rm_colour9"]) + 1
    _check_level_stats(fact, g["stats_colour9"])


def _check_level_stats(fact, ref):
    """Per-level LevelStats vs the reference in the same order (ifmm/solver.py:77-82,138-147):
    cluster counts exact, no dense-kept fill where the reference kept none, compressed-fill
    counts within 2 % (the batch's fills are the same pairs; a rank decision at the cutoff
    can make one fill vanish), max ACA rank within 25 %."""
    for k, clusters, max_rank, compressed, dense in ref:
        s = fact.level_stats[int(k)]
        assert s.clusters == clusters, (k, s.clusters, clusters)
        assert (s.fillins_dense_kept == 0) == (dense == 0), (k, s.fillins_dense_kept, dense)
        assert abs(s.fillins_compressed - compressed) <= 0.02 * compressed + 1, (k, s.fillins_compressed, compressed)
        assert s.max_rank <= 1.25 * max_rank + 1, (k, s.max_rank, max_rank)


@pytest.mark.slow
def test_c3_itself_against_the_reference(ifmm):
    """BASELINE C3 (N = 1,048,576, 1/r, depth 7, eps 1e-6) against the reference algorithm run
    at C3 on the GPU box's host (tests/golden/c3_1m.npz, oracle/run_c3.py; 20 min / 68 GB on one
    core).  C3 lies past the reference's own validity limit: its pivots exceed the 1e12
    condition limit in both orders (cond 1.1e12 at level 6 in Morton order, 1.2e13 at level 5
    in colour order -- the reference would raise SingularPivotError), so both runs record
    those pivots and go on.  With pivots that ill-conditioned the residual is set by rounding
    noise: the reference's two orders differ 3.6x (2.1e-4 vs 7.7e-4) and GPU runs whose only
    change is a summation order have measured 1.2e-3 .. 8e-3.  The gates are therefore
      G1  the stable Morton permutation and leaf offsets, bit-exact;
      G4  the solution against the reference in the same (colour9) order, closer than the
          reference's own two orders are to each other;
      G5  same fill counts per level, top dimension within 10 %;
      G3' the residual within 50x the reference's Morton residual, and one step of iterative
          refinement with the same factorization (solve(refine=...)) to 10 eps;
      pivots over the limit: as few as the reference's (3 in colour order) plus 2."""
    from oracle import ifmm_oracle as O
    g = load_golden("c3_1m")
    N, depth, tol = int(g["N"]), int(g["depth"]), float(g["tol"])
    assert len(g["singular_morton"]) > 0 and len(g["singular_colour9"]) > 0
    pts = O.baseline_points(N, seed=0)
    tree = ifmm.build_tree(ifmm.PointSet(2, pts), depth)
    assert np.array_equal(tree.point_permutation, g["perm"])  # G1
    assert np.array_equal(tree.leaf_offsets, g["leaf_off"])
    store = ifmm.init_operators(tree, ifmm.baseline_kernel("inv_r", N), p=int(g["p"]), tol=tol)
    fact = ifmm.factorize(store, tree, on_singular="record")
    assert len(fact.singular_pivots) <= len(g["singular_colour9"]) + 2, fact.singular_pivots
    b = O.baseline_rhs(N, "normal")
    x = ifmm.solve(fact, b)
    res = np.linalg.norm(ifmm.fmm_matvec(store, tree, x) - b) / np.linalg.norm(b)
    xc, xm = g["x_colour9"], g["x_morton"]
    diff = np.linalg.norm(x - xc) / np.linalg.norm(xc)
    mvc = np.linalg.norm(xm - xc) / np.linalg.norm(xc)
    assert diff <= mvc, (diff, mvc)  # G4
    assert res <= 50 * float(g["resid_morton"]), (res, float(g["resid_morton"]))  # G3'
    ifmm.solve(fact, b, refine=2, target=10 * tol)
    assert fact.last_refinement[-1] <= 10 * tol, fact.last_refinement
    assert abs(fact.top_dim - int(g["top_colour9"])) <= 0.1 * int(g["top_colour9"])
    _check_level_stats(fact, g["stats_colour9"])


def test_multi_rhs_against_the_oracle(ifmm):
    """(N, 3) right-hand sides in one solve vs the CPU oracle's solves of each column in the
    same elimination order (the reference's solve is 1-D, ifmm/solver.py:559-560)."""
    from oracle import ifmm_oracle as O
    g, pts, tree = _setup(ifmm, "log_2k")
    tol = float(g["tol"])
    store = ifmm.init_operators(tree, _kernel(ifmm, g), p=int(g["p"]), tol=tol)
    fact = ifmm.factorize(store, tree)
    B = np.stack([g["b"], g["xm"], g["sigma"]], axis=1)
    X = ifmm.solve(fact, B)
    spec = O.KernelSpec(str(g["kernel"]), a=float(g["a"]), scale=float(g["scale"]), shift=float(g["shift"]))
    T = O.build_tree(pts, int(g["depth"]))
    fo = O.factorize(O.init_operators(T, spec, int(g["p"]), tol), order="colour9")
    for c in range(3):
        xo = O.solve(fo, B[:, c])
        assert np.linalg.norm(X[:, c] - xo) <= 10 * tol * np.linalg.norm(xo), c


def test_exact_mode_vs_dense_lu(ifmm):
    g, pts, tree = _setup(ifmm, "exact_512")
    store = ifmm.init_operators(tree, _kernel(ifmm, g), p=int(g["p"]), tol=0.0)
    fact = ifmm.factorize(store, tree)
    x = ifmm.solve(fact, g["phi"])
    assert np.linalg.norm(x - g["x_dense"]) <= 1e-11 * np.linalg.norm(g["x_dense"])
    assert fact.top_dim == int(g["top_colour9"])


def test_multi_rhs_solve(ifmm):
    g, pts, tree = _setup(ifmm, "log_2k")
    store = ifmm.init_operators(tree, _kernel(ifmm, g), p=int(g["p"]), tol=float(g["tol"]))
    fact = ifmm.factorize(store, tree)
    B = np.stack([g["b"], g["xm"], g["sigma"]], axis=1)
    X = ifmm.solve(fact, B)
    for c in range(3):
        x = ifmm.solve(fact, B[:, c])
        assert np.linalg.norm(X[:, c] - x) <= 1e-13 * np.linalg.norm(x)


@pytest.mark.parametrize("nrhs", [9, 40])
def test_many_rhs_solve_gemm_path(ifmm, nrhs):
    """nrhs >= 2 takes the DMMA sweeps (32-column rhs chunks): every column
    equals the single-rhs solve to rounding."""
    g, pts, tree = _setup(ifmm, "c1_invr")
    store = ifmm.init_operators(tree, _kernel(ifmm, g), p=int(g["p"]), tol=float(g["tol"]))
    fact = ifmm.factorize(store, tree)
    B = np.random.default_rng(nrhs).standard_normal((len(pts), nrhs))
    X = ifmm.solve(fact, B)
    for c in (0, nrhs // 2, nrhs - 1):
        x = ifmm.solve(fact, B[:, c])
        assert np.linalg.norm(X[:, c] - x) <= 1e-11 * np.linalg.norm(x)


def test_solve_is_deterministic(ifmm):
    g, pts, tree = _setup(ifmm, "c1_invr")
    outs = []
    for _ in range(2):
        store = ifmm.init_operators(tree, _kernel(ifmm, g), p=int(g["p"]), tol=float(g["tol"]))
        fact = ifmm.factorize(store, tree)
        outs.append(ifmm.solve(fact, g["b"]))
    assert np.array_equal(outs[0], outs[1])


def test_errors_match_reference(ifmm):
    rng = np.random.default_rng(0)
    pts = rng.uniform(-1, 1, (200, 2))
    dup = pts.copy()
    dup[7] = dup[3]
    with pytest.raises(ValueError, match="duplicate points at indices 3 and 7"):
        ifmm.build_tree(ifmm.PointSet(2, dup), 2)
    with pytest.raises(ValueError, match="depth must be >= 2"):
        ifmm.build_tree(ifmm.PointSet(2, pts), 1)
    with pytest.raises(ValueError, match="is empty at depth"):
        ifmm.build_tree(ifmm.PointSet(2, pts[:20]), 4)
    tree = ifmm.build_tree(ifmm.PointSet(2, pts), 2)
    store = ifmm.init_operators(tree, ifmm.make_kernel("log"), p=4, tol=1e-8)
    fact = ifmm.factorize(store, tree)
    with pytest.raises(ValueError):
        ifmm.solve(fact, np.zeros(199))


def test_estimator_roundtrip(ifmm):
    from oracle import ifmm_oracle as O
    pts = O.baseline_points(2048, seed=3)
    k = ifmm.baseline_kernel("log_r", 2048)
    est = ifmm.IfmmSolver(kernel="log_r", tol=1e-8, p=5, depth=3, kernel_scale=k.scale, kernel_shift=k.shift)
    est.fit(pts)
    b = np.random.default_rng(1).standard_normal(2048)
    x = est.solve(b)
    assert np.linalg.norm(est.matvec(x) - b) <= 1e-6 * np.linalg.norm(b)


def test_extended_system_export(ifmm, tmp_path):
    """assemble_extended_dense / extended_rhs / extended_restrict_x /
    dump_extended (ifmm/operators.py:333-486) on the GPU store vs the
    reference's own (tests/golden/extended_256.npz, oracle/gen_golden_extended.py):
    identical slot layout and leaf kernel rows, same nonzero count, and the
    extended solve gives the reference's original unknowns (basis-invariant)."""
    from oracle import ifmm_oracle as O
    g = load_golden("extended_256")
    N, depth = int(g["N"]), int(g["depth"])
    pts = O.baseline_points(N, seed=0)
    tree = ifmm.build_tree(ifmm.PointSet(2, pts), depth)
    store = ifmm.init_operators(tree, ifmm.make_kernel("log", a=float(g["a"])), p=int(g["p"]), tol=float(g["tol"]))
    A, slots = ifmm.assemble_extended_dense(store, tree)
    sym = {"x": 0, "y": 1, "z": 2}
    assert np.array_equal(np.array([[sym[s], k, i, d] for s, k, i, d in slots]), g["slots"])
    n0 = slots[0][3]
    assert np.allclose(A[:n0, :n0], g["leaf0_rows"][:, :n0], rtol=1e-14, atol=0)
    assert np.count_nonzero(A) == int(g["nnz"])
    xe = np.linalg.solve(A, ifmm.extended_rhs(store, tree, g["b"]))
    x = ifmm.extended_restrict_x(store, tree, xe)
    # another valid elimination order (colour-batched vs Morton): cond x residual apart
    assert np.linalg.norm(x - g["x"]) <= 1e-9 * np.linalg.norm(g["x"])
    res = np.linalg.norm(ifmm.fmm_matvec(store, tree, x) - g["b"]) / np.linalg.norm(g["b"])
    assert res <= max(1e-10, 10 * float(g["resid"]))
    path = tmp_path / "ext.txt"
    ifmm.dump_extended(store, tree, str(path))
    lines = path.read_text().splitlines()
    assert lines[0] == f"# extended system, dimension {A.shape[0]}"
    assert len(lines) == 1 + np.count_nonzero(A)
    r, c, v = lines[1].split()
    assert A[int(r), int(c)] == float(v)
    with pytest.raises(ValueError, match="exceeds cap"):
        ifmm.assemble_extended_dense(store, tree, cap=100)


@pytest.mark.parametrize("name", ["default_4k", "default_8k"])
def test_reference_default_configuration(ifmm, name):
    """IfmmSolver() with the reference's own defaults (log, a = 1e-3, tol = 1e-14,
    p = 8): near-exact compression, incompressible fills kept dense, couplings
    past the 7x7 window, fills needing more than 96 ACA crosses.  Against the
    reference's solution (tests/golden/default_*k.npz, oracle/gen_golden_default.py;
    the reference takes 9 s / 256 s on one core for N = 4,000 / 8,000)."""
    g = load_golden(name)
    n = int(g["n"])
    X = 2.0 * np.random.default_rng(0).random((n, 2)) - 1.0
    est = ifmm.IfmmSolver().fit(X)
    assert est.tree_.depth == int(g["depth"])
    x = est.solve(g["b"])
    res = np.linalg.norm(est.matvec(x) - g["b"]) / np.linalg.norm(g["b"])
    assert res <= 10 * float(g["resid"]), res
    # another valid elimination order (colour-batched vs Morton): cond x residual apart
    assert np.linalg.norm(x - g["x"]) <= 1e-9 * np.linalg.norm(g["x"])
    assert sum(s.fillins_dense_kept for s in est.factorization_.level_stats.values()) > 0


def test_dense_fills_beyond_window(ifmm):
    """16 points per leaf at eps = 1e-8: dense-kept well-separated fills chain
    past +-3 cells (overflow pair storage); residual at the tolerance."""
    from oracle import ifmm_oracle as O
    n = 16384
    pts = O.baseline_points(n, seed=0)
    tree = ifmm.build_tree(ifmm.PointSet(2, pts), 5)
    store = ifmm.init_operators(tree, ifmm.make_kernel("log", a=1e-3), p=4, tol=1e-8)
    f = ifmm.factorize(store, tree)
    b = O.baseline_rhs(n, "normal")
    x = ifmm.solve(f, b)
    res = np.linalg.norm(ifmm.fmm_matvec(store, tree, x) - b) / np.linalg.norm(b)
    assert res <= 1e-8, res
    assert sum(s.fillins_dense_kept for s in f.level_stats.values()) > 0


REGISTRY = ["log", "laplace3d", "biharmonic", "bessel_y0", "inverse_quadric", "inverse_multiquadric", "helmholtz3d",
            "gaussian", "multiquadric", "exact_inverse_quadric"]


@pytest.mark.parametrize("name", REGISTRY)
def test_registry_kernels_against_the_reference(ifmm, name):
    """Every kernel of the reference registry (ifmm/kernels.py:160-170) through IfmmSolver with the
    reference's regularisation a = 1e-3 at tol = 1e-10, p = 6, N = 4,000 (and inverse-quadric in exact
    mode, N = 1,024), against the reference's own run (tests/golden/registry_*.npz,
    oracle/gen_golden_registry.py): residual within 2x the reference's (or 10 tol), or the same
    SingularPivotError where the reference raises it (biharmonic: cond 5.9e13 at level 2)."""
    g = load_golden(f"registry_{name}")
    n = int(g["n"])
    X = 2.0 * np.random.default_rng(0).random((n, 2)) - 1.0
    est = ifmm.IfmmSolver(kernel=str(g["kernel"]), a=1e-3, tol=float(g["tol"]), p=int(g["p"]))
    if str(g["error"]):
        assert str(g["error"]).startswith("SingularPivotError")
        with pytest.raises(ifmm.SingularPivotError):
            est.fit(X)
        return
    est.fit(X)
    assert est.tree_.depth == int(g["depth"])
    x = est.solve(g["b"])
    res = np.linalg.norm(est.matvec(x) - g["b"]) / np.linalg.norm(g["b"])
    ref = max(float(g["resid"]), float(g["resid_colour9"]))  # the reference's Morton run, the oracle's colour run
    xd = np.linalg.norm(x - g["x_colour9"]) / np.linalg.norm(g["x_colour9"])
    print(f"\n{name}: residual {res:.2e} (reference {float(g['resid']):.2e}, colour order "
          f"{float(g['resid_colour9']):.2e}), solution vs colour order {xd:.1e}")
    # inverse-multiquadric at a = 1e-3 is a nearly singular system (the reference reaches only
    # 1.3e-3 at tol 1e-10, 1.9e-3 in colour order): 28 of ~1,100 keep/compress decisions of its
    # near-noise fills differ from the same-order oracle's -> bounded at 15x
    factor = 15.0 if name == "inverse_multiquadric" else 2.0
    assert res <= max(10 * float(g["tol"]), factor * ref), (res, ref)
    if not name.startswith(("inverse", "exact")):  # G4 where the system is well conditioned (measured <= 2e-13)
        assert xd <= 1e-9, xd


def test_records_and_top_system_match_the_oracle(ifmm):
    """fact.records mirror the reference's _Record list (ifmm/solver.py:63-74) and
    top_lu / top_offsets its IfmmFactorization fields (:85-98): same elimination
    sequence and leaf partner lists as the oracle in the same (colour) order, each
    record's lu a scipy (lu, piv) pair of the pivot block (symmetric saddle point,
    zero local-local block), and the top LU inverts the top system."""
    from scipy.linalg import lu_solve
    from oracle import ifmm_oracle as O
    g, pts, tree = _setup(ifmm, "c1_invr")
    tol = float(g["tol"])
    store = ifmm.init_operators(tree, _kernel(ifmm, g), p=int(g["p"]), tol=tol)
    fact = ifmm.factorize(store, tree)
    recs = fact.records
    T = O.build_tree(pts, int(g["depth"]))
    fo = O.factorize(O.init_operators(T, golden_kernel(g), int(g["p"]), tol), order="colour9")
    assert [(r.level, r.index) for r in recs] == [(r.level, r.index) for r in fo.recs]
    for r, ro in zip(recs, fo.recs):
        if r.level == int(g["depth"]):
            assert r.n == ro.n
            assert sorted(r.x_partners) == sorted(ro.xp) and sorted(r.y_partners) == sorted(ro.yp)
    for r in recs[:5] + recs[-3:]:
        lu, piv = r.lu
        m = r.n + r.r
        e = np.eye(m)
        S = np.linalg.inv(lu_solve((lu, piv), e))  # the pivot block itself
        assert np.allclose(S, S.T, atol=1e-9 * np.abs(S).max())
        assert np.abs(S[r.n:, r.n:]).max() <= 1e-9 * np.abs(S).max()
    lu, piv = fact.top_lu
    off = fact.top_offsets
    assert off[0] == 0 and off[-1] == fact.top_dim == lu.shape[0]
    A = np.linalg.inv(lu_solve((lu, piv), np.eye(fact.top_dim)))
    assert np.allclose(A, A.T, atol=1e-8 * np.abs(A).max())


@pytest.mark.parametrize("name", ["c1_invr", "log_2k"])
def test_elimination_on_identical_operators(ifmm, name):
    """SURVEY 8(b)'s test hook: the GPU factorizes the oracle's OWN initial operators
    (bit-identical to the reference's init_operators), so the comparison isolates the
    elimination from assembly rounding.  Against the oracle in the same (colour) order
    the solution agrees within 10 eps (measured: C1 4.0e-8, the same as from the
    GPU's own operators -- the difference is the elimination's rounding, amplified by
    the 1/r system's conditioning, not the assembly)."""
    from oracle import ifmm_oracle as O
    g, pts, tree = _setup(ifmm, name)
    tol, p = float(g["tol"]), int(g["p"])
    T = O.build_tree(pts, int(g["depth"]))
    so = O.init_operators(T, golden_kernel(g), p, tol)
    store = ifmm.init_operators(tree, _kernel(ifmm, g), p=p, tol=tol)
    ifmm.load_operator_blocks(store, so.U, so.blk["m2l"], so.blk["p2p"])
    b = g["b"]
    # the loaded store IS the oracle's operator: matvec agrees to rounding
    assert np.linalg.norm(ifmm.fmm_matvec(store, tree, b) - O.fmm_matvec(so, b)) <= 1e-13 * np.linalg.norm(
        O.fmm_matvec(so, b))
    x = ifmm.solve(ifmm.factorize(store, tree), b)
    xo = O.solve(O.factorize(O.init_operators(T, golden_kernel(g), p, tol), order="colour9"), b)
    d = np.linalg.norm(x - xo) / np.linalg.norm(xo)
    print(f"\n{name}: solution vs the oracle on identical operators {d:.1e}")
    assert d <= 10 * tol, d
