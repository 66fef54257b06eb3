"""GPU unit tests of the batched dense kernels through the C-ABI test hooks,
against numpy/scipy fp64 references."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    from paper_1407_1572_b200 import _lib
    if _lib.lib.ifmm_device_count() == 0:
        pytest.skip("no CUDA device")
    return _lib


@pytest.fixture(params=["cta", "warp"])
def group(request, L):
    """Run the small-matrix hooks CTA-wide or on one warp (fine-level workers)."""
    L.check(L.lib.ifmm_test_set_group(1 if request.param == "warp" else 0))
    yield request.param
    L.check(L.lib.ifmm_test_set_group(0))


@pytest.mark.parametrize("ta,tb,tc", [(0, 0, 0), (1, 0, 0), (0, 1, 0), (1, 1, 1), (1, 0, 1)])
@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (64, 64, 16), (97, 130, 53), (200, 17, 300)])
def test_gemm(L, ta, tb, tc, M, N, K):
    rng = np.random.default_rng(M * 7 + N + K)
    A = rng.standard_normal((K, M) if ta else (M, K))
    B = rng.standard_normal((N, K) if tb else (K, N))
    C0 = rng.standard_normal((N, M) if tc else (M, N))
    Af, Bf, Cf = (np.asfortranarray(x) for x in (A, B, C0))
    C = Cf.copy(order="F")
    L.check(L.lib.ifmm_test_gemm(ta, tb, M, N, K, -0.5, Af.ctypes.data_as(ctypes.c_void_p), Af.shape[0],
                                 Bf.ctypes.data_as(ctypes.c_void_p), Bf.shape[0], 2.0,
                                 C.ctypes.data_as(ctypes.c_void_p), C.shape[0], tc))
    opA = A.T if ta else A
    opB = B.T if tb else B
    ref = -0.5 * opA @ opB + 2.0 * (C0.T if tc else C0)
    got = C.T if tc else C
    assert np.allclose(got, ref, rtol=1e-13, atol=1e-12)


def _saddle(rng, n, r):
    P = rng.standard_normal((n, n))
    P = P + P.T + n * np.eye(n) * 0.1
    U, _ = np.linalg.qr(rng.standard_normal((n, r)))
    S = np.zeros((n + r, n + r))
    S[:n, :n] = P
    S[:n, n:] = U
    S[n:, :n] = U.T
    return S


def _run_lu(L, mats):
    sizes = np.array([m.shape[0] for m in mats], dtype=np.int32)
    packed = np.concatenate([np.asfortranarray(m).ravel(order="F") for m in mats])
    perm = np.zeros(int(sizes.sum()), dtype=np.int32)
    info = np.zeros(len(mats), dtype=np.int32)
    est = np.zeros(len(mats))
    L.check(L.lib.ifmm_test_lu(L.ptr(packed), L.ptr(sizes), len(mats), L.ptr(perm), L.ptr(info), L.ptr(est)))
    out, off, offm = [], 0, 0
    for k in sizes:
        out.append((packed[off:off + k * k].reshape((k, k), order="F"), perm[offm:offm + k]))
        off += k * k
        offm += k
    return out, info, est


def _check_lu(A, LU, perm, tol=1e-13):
    """P A = L U with |L| <= 1 (partial pivoting), backward error ~ eps."""
    k = A.shape[0]
    Lm = np.tril(LU, -1) + np.eye(k)
    Um = np.triu(LU)
    assert sorted(perm.tolist()) == list(range(k))
    assert np.abs(Lm).max() <= 1.0 + 1e-15
    err = np.linalg.norm(A[perm] - Lm @ Um) / (np.linalg.norm(A) * k)
    assert err <= tol, err


def test_lu_batched_variable_sizes(L):
    """Pivot blocks S = [[P, U], [U^T, 0]] of all shapes the factorization meets,
    plus a general matrix; factors, permutation and the dgecon-style estimate of
    ||S^-1||_1 against LAPACK (ifmm/solver.py:214-218)."""
    from scipy.linalg import lu_factor
    from scipy.linalg.lapack import dgecon
    rng = np.random.default_rng(0)
    mats = [_saddle(rng, n, r) for n, r in [(5, 2), (64, 40), (64, 64), (90, 31), (250, 70), (3, 0), (1, 1)]]
    mats.append(rng.standard_normal((700, 700)))
    res, info, est = _run_lu(L, mats)
    assert not info.any()
    for A, (LU, perm), e in zip(mats, res, est):
        _check_lu(A, LU, perm)
        lu_ref = lu_factor(A)
        rc = dgecon(lu_ref[0], np.linalg.norm(A, 1), norm="1")[0]
        exact = np.linalg.norm(np.linalg.inv(A), 1)
        # both estimates are lower bounds of the exact norm and (dlacn2) almost always equal to it
        assert e <= exact * (1 + 1e-10)
        assert e >= 0.3 * exact
        assert abs(e * np.linalg.norm(A, 1) * rc - 1.0) < 0.5


def _saddle_cond(rng, n, r, cond):
    """Saddle-point pivot block whose P2P part has condition number `cond`."""
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    P = Q @ np.diag(np.logspace(0, -np.log10(cond), n)) @ Q.T
    U, _ = np.linalg.qr(rng.standard_normal((n, r)))
    S = np.zeros((n + r, n + r))
    S[:n, :n] = P
    S[:n, n:] = U
    S[n:, :n] = U.T
    return S


@pytest.mark.parametrize("n,r", [(64, 50), (300, 120), (500, 200)])
@pytest.mark.parametrize("cond", [1e6, 1e12, 1e14])
def test_lu_ill_conditioned_matches_lapack(L, n, r, cond):
    """Ill-conditioned pivots (the regime the pivot-condition test guards):
    the condition estimate equals LAPACK dgecon's (same dlacn2 iterates on the
    triangular factors), and X = S^-1 C is backward stable like lu_solve
    (ifmm/solver.py:214-218,246)."""
    from scipy.linalg import lu_factor, lu_solve
    from scipy.linalg.lapack import dgecon
    rng = np.random.default_rng(n + int(np.log10(cond)))
    S = _saddle_cond(rng, n, r, cond)
    res, info, est = _run_lu(L, [S])
    LU, perm = res[0]
    lu = lu_factor(S)
    ref = 1.0 / (dgecon(lu[0], np.linalg.norm(S, 1), norm="1")[0] * np.linalg.norm(S, 1))
    assert abs(est[0] / ref - 1.0) < 1e-6, (est[0], ref)
    wl = 3 * n
    C = np.asfortranarray(rng.standard_normal((n, wl)))
    xt = np.zeros((n, wl + r), order="F")
    xb = np.zeros((r, wl + r), order="F")
    L.check(L.lib.ifmm_test_lu_solve_x(L.ptr(np.asfortranarray(LU)), L.ptr(perm.astype(np.int32)), n, r, L.ptr(C),
                                       wl, L.ptr(xt), L.ptr(xb)))
    Cf = np.zeros((n + r, wl + r))
    Cf[:n, :wl] = C
    Cf[n:, wl:] = -np.eye(r)
    X = np.vstack([xt, xb])
    Xr = lu_solve(lu, Cf)
    be = np.linalg.norm(S @ X - Cf) / (np.linalg.norm(S) * np.linalg.norm(X))
    be_ref = np.linalg.norm(S @ Xr - Cf) / (np.linalg.norm(S) * np.linalg.norm(Xr))
    assert be <= max(4 * be_ref, 1e-15), (be, be_ref)


def test_lu_large_batch_mixed_sizes(L):
    rng = np.random.default_rng(7)
    sizes = [int(x) for x in rng.integers(40, 140, size=80)] + [64, 96, 97, 127, 128, 129]
    mats = [_saddle(rng, max(1, m - m // 3), m // 3) for m in sizes]
    res, info, _ = _run_lu(L, mats)
    assert not info.any()
    for A, (LU, perm) in zip(mats, res):
        _check_lu(A, LU, perm)


@pytest.mark.parametrize("m", [900, 1100, 2500])
def test_lu_large_single(L, m):
    """Single large systems (the level-2 top system): narrower panels above m ~ 830."""
    rng = np.random.default_rng(m)
    A = rng.standard_normal((m, m)) + m ** 0.5 * np.eye(m)
    res, info, _ = _run_lu(L, [A])
    assert info[0] == 0
    _check_lu(A, *res[0])


def test_lu_pivot_order_matches_lapack(L):
    """Same pivot choices as dgetrf (no ties): identical permutation and factors to rounding."""
    from scipy.linalg import lu_factor
    rng = np.random.default_rng(3)
    A = _saddle(rng, 100, 37)
    res, info, _ = _run_lu(L, [A])
    LU, perm = res[0]
    lu_ref, piv = lu_factor(A)
    p = np.arange(A.shape[0])
    for c, q in enumerate(piv):
        p[[c, q]] = p[[q, c]]
    assert np.array_equal(perm, p)
    assert np.allclose(LU, lu_ref, rtol=1e-10, atol=1e-12)


def test_lu_flags_singular(L):
    A = np.zeros((4, 4))
    A[0, 0] = A[1, 1] = 1.0
    _, info, _ = _run_lu(L, [A])
    assert info[0] == 3


@pytest.mark.parametrize("n,r,wl", [(64, 40, 300), (7, 3, 5), (250, 70, 900), (600, 300, 40), (40, 0, 17)])
def test_lu_solve_x(L, n, r, wl):
    """X = S^-1 [[C, 0], [0, -I]] on the coupling panel (ifmm/solver.py:232-246) vs lu_solve."""
    from scipy.linalg import lu_factor, lu_solve
    rng = np.random.default_rng(n + r + wl)
    S = _saddle(rng, n, r)
    m, w = n + r, wl + r
    (LU, perm) = _run_lu(L, [S])[0][0]
    C = np.asfortranarray(rng.standard_normal((n, wl)))
    xt = np.zeros((n, w), order="F")
    xb = np.zeros((r, w), order="F")
    LUf = np.asfortranarray(LU)
    L.check(L.lib.ifmm_test_lu_solve_x(L.ptr(LUf), L.ptr(perm.astype(np.int32)), n, r, L.ptr(C), wl, L.ptr(xt),
                                       L.ptr(xb)))
    Cf = np.zeros((m, w))
    Cf[:n, :wl] = C
    Cf[n:, wl:] = -np.eye(r)
    X = lu_solve(lu_factor(S), Cf)
    assert np.linalg.norm(np.vstack([xt, xb]) - X) <= 1e-11 * np.linalg.norm(X)


@pytest.mark.parametrize("m,n", [(16, 16), (432, 16), (64, 40), (300, 64), (7, 3), (12, 9), (8, 8), (30, 30), (5, 14),
                                 (32, 32), (2, 2), (1, 1)])
def test_jacobi_svd(L, group, m, n):
    rng = np.random.default_rng(m + n)
    A = rng.standard_normal((m, n)) @ np.diag(np.logspace(0, -12, n))
    a = np.asfortranarray(A).copy(order="F")
    V = np.empty((n, n), order="F")
    sig = np.empty(n)
    L.check(L.lib.ifmm_test_jacobi(L.ptr(a), m, n, L.ptr(V), L.ptr(sig)))
    s_ref = np.linalg.svd(A, compute_uv=False)
    s_got = np.sort(sig)[::-1]
    assert np.allclose(s_got[:len(s_ref)], s_ref, rtol=1e-9, atol=1e-14 * s_ref[0])
    assert np.all(s_got[len(s_ref):] <= 1e-12 * s_ref[0])  # m < n: the extra columns are rotated to zero
    assert np.allclose(a, A @ V, atol=1e-12 * s_ref[0])
    assert np.allclose(V.T @ V, np.eye(n), atol=1e-12)


@pytest.mark.parametrize("m,k", [(10, 3), (100, 16), (500, 64), (16, 16)])
def test_householder_qr(L, group, m, k):
    rng = np.random.default_rng(m * k)
    A = rng.standard_normal((m, k))
    Q = np.empty((m, k), order="F")
    R = np.empty((k, k), order="F")
    L.check(L.lib.ifmm_test_qr(L.ptr(np.asfortranarray(A)), m, k, L.ptr(Q), L.ptr(R)))
    assert np.allclose(Q @ R, A, atol=1e-12)
    assert np.allclose(Q.T @ Q, np.eye(k), atol=1e-12)
    assert np.allclose(np.tril(R, -1), 0)


@pytest.mark.parametrize("m,n,rank", [(40, 60, 5), (16, 120, 12), (200, 150, 30)])
def test_aca_matches_oracle_crosses(L, group, m, n, rank):
    from oracle import ifmm_oracle as O
    rng = np.random.default_rng(m + n)
    F = rng.standard_normal((m, rank)) @ rng.standard_normal((rank, n)) * np.logspace(0, -6, n)
    probes = L.aca_probe_row(m)
    kmax = min(m, n)
    left = np.empty((m, kmax), order="F")
    right = np.empty((n, kmax), order="F")
    rk = np.zeros(1, dtype=np.int32)
    inc = np.zeros(1, dtype=np.int32)
    L.check(L.lib.ifmm_test_aca(L.ptr(np.asfortranarray(F)), m, n, 1e-8, L.ptr(probes), kmax,
                                L.ptr(left), L.ptr(right), L.ptr(rk), L.ptr(inc)))
    k = int(rk[0])
    approx = left[:, :k] @ right[:, :k].T
    assert np.linalg.norm(approx - F) <= 1e-6 * np.linalg.norm(F)
    Lo, Ro, bad = O.aca_block(F, 1e-8)
    assert not bad and not inc[0]
    assert abs(k - Lo.shape[1]) <= 2


@pytest.mark.parametrize("m,n,seed", [(30, 40, 1), (90, 60, 2), (240, 200, 3)])
def test_aca_random_restarts_match_the_reference(L, group, m, n, seed):
    """Two uncoupled low-rank blocks separated by zero rows: once the first block is
    exhausted ACA meets zero pivots and restarts from random unused rows
    (ifmm/lowrank.py:224-226).  The device draws them from the same PCG64 stream
    (probe-table state + Generator.integers' bounded draw), so the crosses are the
    oracle's (= the reference's) row for row -- restarting at the lowest unused row
    instead finds 3 crosses where the reference finds 7."""
    from oracle import ifmm_oracle as O
    rng = np.random.default_rng(seed)
    q = m // 3
    F = np.zeros((m, n))
    F[:q, :n // 2] = rng.standard_normal((q, 3)) @ rng.standard_normal((3, n // 2))
    F[2 * q:, n // 2:] = rng.standard_normal((m - 2 * q, 4)) @ rng.standard_normal((4, n - n // 2))
    probes = L.aca_probe_row(m)
    kmax = min(m, n)
    left = np.zeros((m, kmax), order="F")
    right = np.zeros((n, kmax), order="F")
    rk = np.zeros(1, dtype=np.int32)
    inc = np.zeros(1, dtype=np.int32)
    L.check(L.lib.ifmm_test_aca(L.ptr(np.asfortranarray(F)), m, n, 1e-8, L.ptr(probes), kmax, L.ptr(left),
                                L.ptr(right), L.ptr(rk), L.ptr(inc)))
    k = int(rk[0])
    Lo, Ro = O.aca_crosses(F, 1e-8)
    assert k == Lo.shape[1] > 0, (k, Lo.shape[1])
    assert np.allclose(left[:, :k], Lo, rtol=1e-12, atol=1e-12 * np.abs(Lo).max())
    assert np.allclose(right[:, :k], Ro, rtol=1e-12, atol=1e-12 * np.abs(Ro).max())


@pytest.mark.parametrize("m,n,rank,decay", [(64, 64, 8, 1e-3), (90, 40, 12, 1e-5), (200, 150, 20, 1e-2),
                                            (16, 120, 5, 1e-7), (64, 64, 30, 1e-1)])
def test_fill_recompression_gram_vs_householder(L, m, n, rank, decay):
    """K1 (ACA + recompression) on one fill: the Gram/Cholesky path and the
    Householder path truncate to the same rank and approximate F to the
    tolerance; the kept singular values match numpy's SVD of F."""
    from oracle import ifmm_oracle as O
    rng = np.random.default_rng(m * n + rank)
    s = np.logspace(0, np.log10(decay), rank)
    F = (rng.standard_normal((m, rank)) * s) @ rng.standard_normal((rank, n))
    probes = L.aca_probe_row(m)
    tol = 1e-6
    out = {}
    for gram in (1, 0):
        kf = min(96, m, n)
        left = np.zeros((m, kf), order="F")
        right = np.zeros((n, kf), order="F")
        sv = np.zeros(kf)
        rk = np.zeros(1, dtype=np.int32)
        st = np.zeros(1, dtype=np.int32)
        L.check(L.lib.ifmm_test_recompress(L.ptr(np.asfortranarray(F)), m, n, tol,
                                           L.ptr(probes), gram, L.ptr(left), L.ptr(right),
                                           L.ptr(sv), L.ptr(rk), L.ptr(st)))
        r = int(rk[0])
        assert st[0] == 0
        approx = left[:, :r] @ right[:, :r].T
        assert np.linalg.norm(approx - F) <= 10 * tol * np.linalg.norm(F)
        # right factor orthonormal, left = U * sigma
        assert np.allclose(right[:, :r].T @ right[:, :r], np.eye(r), atol=1e-10)
        out[gram] = (r, sv[:r].copy())
    (rg, sg), (rh, sh) = out[1], out[0]
    assert rg == rh
    s_ref = np.linalg.svd(F, compute_uv=False)[:rg]
    # the ACA stops at the tolerance: singular values within ~tol * sigma_1
    assert np.allclose(sg, s_ref, rtol=1e-6, atol=10 * tol * s_ref[0])
    # both paths recompress the same crosses
    assert np.allclose(sg, sh, rtol=1e-9, atol=1e-10 * s_ref[0])
