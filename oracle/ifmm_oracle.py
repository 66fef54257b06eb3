"""CPU oracle for the IFMM factorize/solve hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy/scipy restatement of the reference package's algorithm
(`/root/reference/pkg/src/ifmm`, cited below as `ifmm/<file>.py:<line>`).  It is
the checker, never the product: only `tests/`, `__graft_entry__.smoke()` and
`bench.py` (cpu_baseline leg and `--impl reference` arm) may import it.  The
product path (`ifmm_b200`) never imports or calls anything here and fails
loudly when its CUDA library is missing.

Parity pin: `oracle/gen_golden.py` runs the real reference (importable in the
build container only) on seeded inputs and stores its outputs under
`tests/golden/`; `tests/test_oracle_golden.py` checks this restatement against
them (tree/lists bit-exact, operators and solutions to rounding).

The restatement keeps the reference's data model (dict of dense blocks in both
orientations, lazily zero-padded) so rounding behaviour follows it closely,
and adds exactly one degree of freedom: the elimination ORDER inside a level.
`order="morton"` is the reference (`ifmm/solver.py:136-137`); `order="colour9"`
is the order the GPU executes (clusters grouped by (gx mod 3, gy mod 3),
Morton order inside each colour).  Because same-colour clusters are >= 3 cells
apart, their neighbourhoods are disjoint and the GPU's batched elimination of
one colour equals this sequential sweep.

Two code paths here are NOT reference behaviour and therefore PARITY UNPINNED
(the reference has no output to pin them to): `factorize(..., rank_tol=)` /
`_consolidate` (rank-growth control; the reference never calls its
`_maybe_consolidate`, ifmm/solver.py:437-492) and `build_tree(...,
allow_empty=True)` with the full-rank absorption rule of the squeeze functions
(the reference raises on an empty leaf, ifmm/geometry.py:191-195).  Both are off
by default, restate the GPU extensions of the same names on the CPU, and are
checked against dense LU where that is possible (tests/test_oracle_golden.py).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
from scipy.linalg import lu_factor, lu_solve, qr, svd
from scipy.linalg.lapack import dgecon

BOX = 1.0               # ifmm/geometry.py:30
DUP_TOL = 1e-14         # ifmm/geometry.py:31
COND_LIMIT = 1e12       # ifmm/solver.py:50


# --------------------------------------------------------------------------
# kernels  (ifmm/kernels.py:26-170) plus the two BASELINE kernels
# --------------------------------------------------------------------------
@dataclass(frozen=True)
class KernelSpec:
    """Radial kernel f(r).  `scale`/`shift` only apply to inv_r / log_r:
    inv_r: scale/r ; log_r: scale*(ln r + shift).  Regularised kernels follow
    ifmm/kernels.py:50-157 (inner branch for 0<r<a, f(0)=0)."""
    name: str
    a: float = 0.001
    scale: float = 1.0
    shift: float = 0.0

    def __call__(self, r):
        return kernel_eval(self, np.asarray(r, dtype=float))


def _two_branch(r, a, inner, outer):
    # ifmm/kernels.py:50-65: inner on 0<r<a, outer on r>=a, 0 at r=0
    r = np.atleast_1d(r)
    out = np.zeros_like(r)
    lo = (r > 0) & (r < a)
    hi = r >= a
    if lo.any():
        out[lo] = inner(r[lo])
    if hi.any():
        out[hi] = outer(r[hi])
    return out


def kernel_eval(spec: KernelSpec, r: np.ndarray) -> np.ndarray:
    a, nm = spec.a, spec.name
    if nm == "inv_r":
        with np.errstate(divide="ignore"):
            return np.where(r > 0, spec.scale / np.where(r > 0, r, 1.0), 0.0)
    if nm == "log_r":
        with np.errstate(divide="ignore"):
            return np.where(r > 0, spec.scale * (np.log(np.where(r > 0, r, 1.0)) + spec.shift), 0.0)
    if nm == "log":  # :68-77
        return _two_branch(r, a, lambda s: s * (np.log(s) - 1) / (a * (np.log(a) - 1)),
                           lambda s: np.log(s) / np.log(a))
    if nm == "laplace3d":  # :80-84
        return _two_branch(r, a, lambda s: s / a, lambda s: a / s)
    if nm == "biharmonic":  # :87-96
        return _two_branch(r, a, lambda s: s**3 * (3 * np.log(s) - 1) / (a**3 * (3 * np.log(a) - 1)),
                           lambda s: s**2 * np.log(s) / (a**2 * np.log(a)))
    if nm == "bessel-y0":  # :99-108
        from scipy.special import y0
        return _two_branch(r, a, lambda s: (1 + y0(a)) / (1 + y0(s)), lambda s: y0(s) / y0(a))
    if nm == "inverse-quadric":  # :111-120
        return _two_branch(r, a, lambda s: np.arctan(s) / np.arctan(a), lambda s: (1 + a**2) / (1 + s**2))
    if nm == "inverse-multiquadric":  # :123-132
        return _two_branch(r, a, lambda s: np.arcsinh(s) / np.arcsinh(a),
                           lambda s: np.sqrt((1 + a**2) / (1 + s**2)))
    if nm == "helmholtz3d":  # :135-140
        return _two_branch(r, a, lambda s: s / a, lambda s: a * np.cos(s) / (s * np.cos(a)))
    if nm == "gaussian":  # :143-148
        return np.exp(-np.atleast_1d(r) ** 2 / a)
    if nm == "multiquadric":  # :151-156
        return np.sqrt(1 + np.atleast_1d(r) ** 2 / a**2)
    raise ValueError(f"unknown kernel {nm!r}")


def kblock(spec, t, s):
    """K(|t_i - s_j|) -- ifmm/kernels.py:189-194."""
    d = np.atleast_2d(t)[:, None, :] - np.atleast_2d(s)[None, :, :]
    return kernel_eval(spec, np.sqrt(np.sum(d * d, axis=2)))


# --------------------------------------------------------------------------
# tree and lists  (ifmm/geometry.py:124-262)
# --------------------------------------------------------------------------
def morton(grid, bits):
    """x bit least significant (ifmm/geometry.py:124-131)."""
    g = np.asarray(grid, dtype=np.int64)
    out = np.zeros(len(g), dtype=np.int64)
    for b in range(bits):
        for ax in range(g.shape[1]):
            out |= ((g[:, ax] >> b) & 1) << (b * g.shape[1] + ax)
    return out


def unmorton(codes, dim, bits):
    c = np.asarray(codes, dtype=np.int64)
    g = np.zeros((len(c), dim), dtype=np.int64)
    for b in range(bits):
        for ax in range(dim):
            g[:, ax] |= ((c >> (b * dim + ax)) & 1) << b
    return g


@dataclass
class Tree:
    depth: int
    dim: int
    points: np.ndarray          # Morton-permuted
    perm: np.ndarray            # permuted position -> original index
    leaf_off: np.ndarray        # (4^depth + 1,)
    grid: dict                  # k -> (4^k, dim) int
    nbr: dict                   # k -> list of sorted lists (self included)
    ilist: dict                 # k -> list of sorted lists
    sparse: bool = False        # built with allow_empty (extension): leaf cells may hold no points

    def n_clusters(self, k):
        return 1 << (self.dim * k)

    def center(self, k, i):
        w = 2.0 * BOX / (1 << k)
        return -BOX + (self.grid[k][i] + 0.5) * w

    def half(self, k):
        return BOX / (1 << k)

    def leaf_pts(self, i):
        return self.points[self.leaf_off[i]:self.leaf_off[i + 1]]

    def range(self, k, i):
        step = 1 << (self.dim * (self.depth - k))
        return int(self.leaf_off[i * step]), int(self.leaf_off[(i + 1) * step])


def check_points(points):
    """PointSet validation (ifmm/geometry.py:47-61)."""
    from scipy.spatial import cKDTree
    pts = np.ascontiguousarray(points, dtype=float)
    if pts.ndim != 2 or pts.shape[1] not in (1, 2, 3):
        raise ValueError("bad point array shape")
    if np.abs(pts).max(initial=0.0) > BOX:
        raise ValueError("point outside the reference box [-1, 1]^d")
    if len(pts) > 1:
        pairs = cKDTree(pts).query_pairs(DUP_TOL)
        if pairs:
            i, j = sorted(pairs)[0]
            raise ValueError(f"duplicate points at indices {i} and {j}")
    return pts


def build_tree(points, depth, allow_empty=False) -> Tree:
    """ifmm/geometry.py:174-226 and compute_lists :229-262.  allow_empty (extension, NOT
    reference behaviour -- the reference raises, ifmm/geometry.py:191-195): accept leaf cells
    without points; the checker of the GPU's build_tree(allow_empty_leaves=True)."""
    pts = check_points(points)
    if depth < 2:
        raise ValueError("depth must be >= 2")
    dim = pts.shape[1]
    side = 1 << depth
    w = 2.0 * BOX / side
    cell = np.floor((pts + BOX) / w).astype(np.int64)
    np.clip(cell, 0, side - 1, out=cell)
    codes = morton(cell, depth)
    perm = np.argsort(codes, kind="stable")
    cnt = np.bincount(codes[perm], minlength=1 << (dim * depth))
    if cnt.min() == 0 and not allow_empty:
        raise ValueError(f"leaf cell {int(np.argmin(cnt))} is empty at depth {depth}")
    off = np.concatenate([[0], np.cumsum(cnt)])
    grid, nbr, il = {}, {}, {}
    shifts = np.stack(np.meshgrid(*([[-1, 0, 1]] * dim), indexing="ij"), -1).reshape(-1, dim)
    for k in range(1, depth + 1):
        g = unmorton(np.arange(1 << (dim * k)), dim, k)
        grid[k] = g
        lst = []
        for i in range(len(g)):
            cand = g[i] + shifts
            ok = np.all((cand >= 0) & (cand < (1 << k)), axis=1)
            lst.append(sorted(int(m) for m in morton(cand[ok], k)))
        nbr[k] = lst
    for k in range(1, depth + 1):
        out = []
        for i in range(1 << (dim * k)):
            if k == 1:
                out.append([])
                continue
            s = set(nbr[k][i])
            cand = [c for pn in nbr[k - 1][i >> dim] for c in range(pn << dim, (pn + 1) << dim)]
            out.append(sorted(c for c in cand if c not in s))
        il[k] = out
    t = Tree(depth, dim, pts[perm], perm, off, grid, nbr, il)
    t.sparse = bool(allow_empty)
    return t


def elimination_order(tree: Tree, k: int, order: str):
    """Elimination order of level k.  morton: ifmm/solver.py:136.  colour9:
    colour c = (gx mod 3) + 3 (gy mod 3) [+ 9 (gz mod 3)], Morton inside a colour."""
    n = tree.n_clusters(k)
    if order == "morton":
        return [list(range(n))]
    g = tree.grid[k]
    col = np.zeros(n, dtype=np.int64)
    for ax in range(tree.dim):
        col += (g[:, ax] % 3) * (3 ** ax)
    return [list(np.nonzero(col == c)[0]) for c in range(3 ** tree.dim) if np.any(col == c)]


# --------------------------------------------------------------------------
# low rank  (ifmm/lowrank.py:56-271)
# --------------------------------------------------------------------------
def cheb1(p):
    return -np.cos((2 * np.arange(p) + 1) * np.pi / (2 * p))


def lagrange(x, nodes):
    L = np.ones((len(x), len(nodes)))
    for j in range(len(nodes)):
        for m in range(len(nodes)):
            if m != j:
                L[:, j] *= (x - nodes[m]) / (nodes[j] - nodes[m])
    return L


def tnodes(center, half, p, dim):
    g = np.meshgrid(*([cheb1(p)] * dim), indexing="ij")
    return np.asarray(center) + half * np.stack([a.ravel() for a in g], axis=1)


def tinterp(pts, center, half, p):
    pts = np.atleast_2d(pts)
    dim = pts.shape[1]
    n1 = cheb1(p)
    out = lagrange((pts[:, 0] - center[0]) / half, n1)
    for d in range(1, dim):
        out = (out[:, :, None] * lagrange((pts[:, d] - center[d]) / half, n1)[:, None, :]).reshape(len(pts), -1)
    return out


def trunc_rank(s, tol):
    """ifmm/lowrank.py:137-144."""
    if len(s) == 0 or s[0] == 0.0:
        return 0
    if tol <= 0:
        return len(s)
    below = np.nonzero(s / s[0] < tol)[0]
    return int(below[0]) if len(below) else len(s)


def tsvd(block, tol):
    """(left*s, right) -- ifmm/lowrank.py:147-161."""
    if block.size == 0:
        return np.zeros((block.shape[0], 0)), np.zeros((block.shape[1], 0))
    U, s, Vt = svd(block, full_matrices=False, lapack_driver="gesdd")
    r = trunc_rank(s, tol)
    return U[:, :r] * s[:r], Vt[:r].T


def recompress(L, R, tol):
    """ifmm/lowrank.py:164-171."""
    if L.shape[1] == 0:
        return L, R
    Ql, Rl = qr(L, mode="economic")
    Qr, Rr = qr(R, mode="economic")
    a, b = tsvd(Rl @ Rr.T, tol)
    return Ql @ a, Qr @ b


def aca_probe_rows(m):
    """The seeded probe-row draw of ifmm/lowrank.py:196-197 (also used by the
    product, which receives this table from its host layer)."""
    rng = np.random.default_rng(0)
    return rng, rng.choice(m, size=min(10, m), replace=False)


def aca_block(F, tol):
    """Partially pivoted ACA + recompression on a dense block.
    Returns (left, right, incompressible).  ifmm/lowrank.py:174-271."""
    m, n = F.shape
    if m == 0 or n == 0:
        return np.zeros((m, 0)), np.zeros((n, 0)), False
    U, V, done = _aca_raw(F, tol)
    if U.shape[1] == 0:
        return np.zeros((m, 0)), np.zeros((n, 0)), False
    L, R = recompress(U, V, tol)
    return L, R, (not done and U.shape[1] >= min(m, n) and tol > 0)


def aca_crosses(F, tol):
    """The raw ACA crosses (u_t, v_t as columns) before recompression."""
    U, V, _ = _aca_raw(F, tol)
    return U, V


def _aca_raw(F, tol):
    """ifmm/lowrank.py:174-263: (crosses U, V, converged)."""
    m, n = F.shape
    full = min(m, n)
    rng, probes = aca_probe_rows(m)
    nxt = max((int(i) for i in probes), key=lambda i: np.abs(F[i]).max(initial=0.0))
    us, vs = [], []
    rows_used, cols_used = set(), set()
    nsq = 0.0
    strikes = 0
    done = False
    while len(us) < full:
        i = nxt
        rows_used.add(i)
        rr = F[i].copy()
        for u, v in zip(us, vs):
            rr -= u[i] * v
        if cols_used:
            rr[list(cols_used)] = 0.0
        j = int(np.argmax(np.abs(rr)))
        piv = rr[j]
        tiny = 1e-15 * np.sqrt(nsq) if nsq > 0 else 1e-300
        if abs(piv) <= tiny:
            strikes += 1
            if strikes >= 3 or len(rows_used) >= m:
                done = True
                break
            nxt = int(rng.choice([r for r in range(m) if r not in rows_used]))
            continue
        strikes = 0
        cols_used.add(j)
        cc = F[:, j].copy()
        for u, v in zip(us, vs):
            cc -= v[j] * u
        u = cc / piv
        v = rr
        csq = float(np.dot(u, u) * np.dot(v, v))
        if us:
            nsq += csq + 2.0 * float(np.abs(np.array([np.dot(u, x) for x in us]))
                                     @ np.abs(np.array([np.dot(v, x) for x in vs])))
        else:
            nsq = csq
        us.append(u)
        vs.append(v)
        if tol > 0 and csq <= tol * tol * nsq:
            done = True
            break
        ua = np.abs(u)
        ua[list(rows_used)] = -1.0
        nxt = int(np.argmax(ua))
        if ua[nxt] < 0:
            done = True
            break
    if not us:
        return np.zeros((m, 0)), np.zeros((n, 0)), done
    return np.stack(us, 1), np.stack(vs, 1), done


# --------------------------------------------------------------------------
# operator store  (ifmm/operators.py:42-274)
# --------------------------------------------------------------------------
class Blocks:
    """Block-sparse extended system: both orientations kept, lazily padded
    (ifmm/operators.py:42-137)."""

    KINDS = ("p2p", "m2l", "p2l", "m2p")

    def __init__(self, tree, spec, p, tol):
        self.tree, self.spec, self.p, self.tol = tree, spec, p, tol
        self.U = {}
        self.blk = {kd: {} for kd in self.KINDS}
        self.pp = {}   # (k,i) -> set j   p2p partners
        self.plr = {}  # (k,i) -> set j with p2l(k,i,j)
        self.plc = {}  # (k,j) -> set i with p2l(k,i,j)
        self.coff = {}
        self.max_init_rank = 0

    def r(self, k, i):
        return self.U[(k, i)].shape[1]

    def n(self, k, i):
        return self.U[(k, i)].shape[0]

    def shape(self, kd, k, i, j):
        a = self.n(k, i) if kd in ("p2p", "m2p") else self.r(k, i)
        b = self.n(k, j) if kd in ("p2p", "p2l") else self.r(k, j)
        return a, b

    def get(self, kd, k, i, j):
        sh = self.shape(kd, k, i, j)
        b = self.blk[kd].get((k, i, j))
        if b is None:
            return np.zeros(sh)
        if b.shape != sh:
            o = np.zeros(sh)
            o[:b.shape[0], :b.shape[1]] = b
            self.blk[kd][(k, i, j)] = o
            return o
        return b

    def add(self, kd, k, i, j, d):
        st = self.blk[kd]
        b = st.get((k, i, j))
        if b is None:
            st[(k, i, j)] = d.copy()
        elif b.shape == d.shape:
            b += d
        else:
            sh = (max(b.shape[0], d.shape[0]), max(b.shape[1], d.shape[1]))
            o = np.zeros(sh)
            o[:b.shape[0], :b.shape[1]] = b
            o[:d.shape[0], :d.shape[1]] += d
            st[(k, i, j)] = o
        if kd == "p2p":
            self.pp.setdefault((k, i), set()).add(j)
            self.pp.setdefault((k, j), set()).add(i)
        elif kd == "p2l":
            self.plr.setdefault((k, i), set()).add(j)
            self.plc.setdefault((k, j), set()).add(i)
        elif kd == "m2p":
            self.plr.setdefault((k, j), set()).add(i)
            self.plc.setdefault((k, i), set()).add(j)

    def drop_hybrid(self, k, p, q):
        self.blk["p2l"].pop((k, p, q), None)
        self.blk["m2p"].pop((k, q, p), None)
        self.plr.get((k, p), set()).discard(q)
        self.plc.get((k, q), set()).discard(p)

    def drop_p2p(self, k, p, q):
        self.blk["p2p"].pop((k, p, q), None)
        self.blk["p2p"].pop((k, q, p), None)
        self.pp.get((k, p), set()).discard(q)
        self.pp.get((k, q), set()).discard(p)

    def refresh_offsets(self, k, i):
        d = self.tree.dim
        dims = [self.r(k + 1, c) for c in range((i << d), (i + 1) << d)]
        self.coff[(k, i)] = np.concatenate([[0], np.cumsum(dims)]).astype(int)


def child_transfers(dim, p):
    """ifmm/operators.py:145-161."""
    n1 = cheb1(p)
    g = np.stack([a.ravel() for a in np.meshgrid(*([n1] * dim), indexing="ij")], axis=1)
    out = []
    for c in range(1 << dim):
        off = np.array([(c >> ax) & 1 for ax in range(dim)], dtype=float) - 0.5
        out.append(tinterp(off + 0.5 * g, np.zeros(dim), 1.0, p))
    return out


def init_operators(tree: Tree, spec: KernelSpec, p=8, tol=1e-14) -> Blocks:
    """ifmm/operators.py:164-274."""
    st = Blocks(tree, spec, p, tol)
    K, d = tree.depth, tree.dim
    if tol == 0.0:
        for k in range(K, 1, -1):
            for i in range(tree.n_clusters(k)):
                lo, hi = tree.range(k, i)
                st.U[(k, i)] = np.eye(hi - lo)
        for k in range(2, K + 1):
            for i in range(tree.n_clusters(k)):
                lo, hi = tree.range(k, i)
                for j in tree.ilist[k][i]:
                    if j < i:
                        continue
                    l2, h2 = tree.range(k, j)
                    b = kblock(spec, tree.points[lo:hi], tree.points[l2:h2])
                    st.add("m2l", k, i, j, b)
                    st.add("m2l", k, j, i, b.T.copy())
    else:
        nd = p ** d
        tr = child_transfers(d, p)
        raw = {}
        for k in range(K, 1, -1):
            nc = tree.n_clusters(k)
            nodes = [tnodes(tree.center(k, i), tree.half(k), p, d) for i in range(nc)]
            for i in range(nc):
                il = tree.ilist[k][i]
                if k == K:
                    lp = tree.leaf_pts(i)
                    B = tinterp(lp, tree.center(k, i), tree.half(k), p) if len(lp) else np.zeros((0, nd))
                else:
                    B = np.concatenate([raw[(k + 1, c)] @ tr[c - (i << d)]
                                        for c in range((i << d), (i + 1) << d)], axis=0)
                ni = B.shape[0]
                if ni == 0:  # an empty cluster (sparse trees): no unknowns
                    st.U[(k, i)] = np.zeros((0, 0))
                    raw[(k, i)] = np.zeros((0, nd))
                    continue
                row = (np.concatenate([kblock(spec, nodes[i], nodes[j]) for j in il], axis=1)
                       if il else np.zeros((nd, 0)))
                Uf, s, _ = svd(row, full_matrices=False)
                keep = min(int(np.sum(s >= (s[0] if len(s) else 0) * tol)), ni, nd)
                Uc, sc, _ = svd(B @ Uf[:, :keep], full_matrices=False)
                ri = int(np.sum(sc >= (sc[0] if len(sc) else 0) * 1e-14))
                st.U[(k, i)] = Uc[:, :ri]
                raw[(k, i)] = Uc[:, :ri].T @ B
                st.max_init_rank = max(st.max_init_rank, ri)
            for i in range(nc):
                for j in tree.ilist[k][i]:
                    if j < i:
                        continue
                    b = raw[(k, i)] @ kblock(spec, nodes[i], nodes[j]) @ raw[(k, j)].T
                    st.add("m2l", k, i, j, b)
                    st.add("m2l", k, j, i, b.T.copy())
    # leaf near field, unit diagonal (ifmm/operators.py:180-194)
    for i in range(tree.n_clusters(K)):
        for j in tree.nbr[K][i]:
            if j < i:
                continue
            b = kblock(spec, tree.leaf_pts(i), tree.leaf_pts(j))
            if j == i:
                np.fill_diagonal(b, 1.0)
                st.add("p2p", K, i, i, b)
            else:
                st.add("p2p", K, i, j, b)
                st.add("p2p", K, j, i, b.T.copy())
    for k in range(1, K):
        for i in range(tree.n_clusters(k)):
            st.refresh_offsets(k, i)
    return st


def fmm_matvec(st: Blocks, x):
    """Compressed forward operator on an un-eliminated store (ifmm/operators.py:282-330)."""
    tree = st.tree
    x = np.asarray(x, dtype=float)
    if x.shape[0] != len(tree.points):
        raise ValueError("charge vector length mismatch")
    xp = x[tree.perm]
    K, d = tree.depth, tree.dim
    y = {}
    for k in range(K, 1, -1):
        for i in range(tree.n_clusters(k)):
            xi = xp[tree.leaf_off[i]:tree.leaf_off[i + 1]] if k == K else \
                np.concatenate([y[(k + 1, c)] for c in range(i << d, (i + 1) << d)])
            y[(k, i)] = st.U[(k, i)].T @ xi
    z = {}
    for k in range(2, K + 1):
        for i in range(tree.n_clusters(k)):
            zi = np.zeros(st.r(k, i))
            for j in tree.ilist[k][i]:
                zi += st.blk["m2l"][(k, i, j)] @ y[(k, j)]
            if k > 2:
                par = i >> d
                o = st.coff[(k - 1, par)]
                c = i - (par << d)
                zi += st.U[(k - 1, par)][o[c]:o[c + 1], :] @ z[(k - 1, par)]
            z[(k, i)] = zi
    out = np.zeros_like(xp)
    for i in range(tree.n_clusters(K)):
        lo, hi = tree.leaf_off[i], tree.leaf_off[i + 1]
        acc = st.U[(K, i)] @ z[(K, i)]
        for j in tree.nbr[K][i]:
            acc = acc + st.blk["p2p"][(K, i, j)] @ xp[tree.leaf_off[j]:tree.leaf_off[j + 1]]
        out[lo:hi] = acc
    res = np.empty_like(out)
    res[tree.perm] = out
    return res


def dense_matrix(spec, points):
    """Identity-plus-kernel system in original point order (ifmm/kernels.py:197-207)."""
    A = kblock(spec, points, points)
    np.fill_diagonal(A, 1.0)
    return A


# --------------------------------------------------------------------------
# factorization  (ifmm/solver.py:106-546)
# --------------------------------------------------------------------------
class SingularPivot(RuntimeError):
    def __init__(self, level, index, cond):
        super().__init__(f"pivot for cluster {index} at level {level} is numerically singular "
                         f"(condition estimate {cond:.2e})")
        self.level, self.index = level, index


@dataclass
class Rec:
    level: int
    index: int
    lu: tuple
    n: int
    r: int
    xp: list
    yp: list


@dataclass
class Stats:
    clusters: int = 0
    max_rank: int = 0
    compressed: int = 0
    dense_kept: int = 0
    aca_ranks: list = field(default_factory=list)


@dataclass
class Factor:
    st: Blocks
    tree: Tree
    tol: float
    recs: list = field(default_factory=list)
    top_lu: tuple = None
    top_off: np.ndarray = None
    stats: dict = field(default_factory=dict)
    r_m: int = 0
    order: str = "morton"
    cond_limit: float = COND_LIMIT
    on_singular: str = "raise"      # "record": note the violation and continue (C3 study)
    singular: list = field(default_factory=list)
    max_cond: dict = field(default_factory=dict)
    rank_control: list = field(default_factory=lambda: [0, 0])  # extension: rank sums before / after


def _parent_near(st: Blocks, k):
    """Level-k P2P from level-(k+1) M2L (ifmm/solver.py:163-192)."""
    tree, d = st.tree, st.tree.dim
    for i in range(tree.n_clusters(k)):
        st.refresh_offsets(k, i)
    for i in range(tree.n_clusters(k)):
        ro = st.coff[(k, i)]
        for j in tree.nbr[k][i]:
            if j < i:
                continue
            co = st.coff[(k, j)]
            b = np.zeros((ro[-1], co[-1]))
            hit = False
            for a in range(1 << d):
                for bb in range(1 << d):
                    sub = st.blk["m2l"].get((k + 1, (i << d) + a, (j << d) + bb))
                    if sub is not None:
                        b[ro[a]:ro[a] + sub.shape[0], co[bb]:co[bb] + sub.shape[1]] = sub
                        hit = True
            if hit:
                st.add("p2p", k, i, j, b)
                if j != i:
                    st.add("p2p", k, j, i, b.T.copy())


def _new_dirs(weight, fac, U, tol, scale):
    """ifmm/solver.py:334-358."""
    cap = U.shape[0] - U.shape[1]
    if cap <= 0 or fac.shape[1] == 0:
        return np.zeros((U.shape[0], 0))
    res = fac - U @ (U.T @ fac)
    res -= U @ (U.T @ res)
    _, s, Vt = svd(weight @ res.T, full_matrices=False)
    w = min(int(np.sum(s > (tol if tol > 0 else 1e-13) * scale)), cap)
    W = Vt[:w].T
    if w:
        W -= U @ (U.T @ W)
    return W


def _augment(st: Blocks, k, q, W):
    """ifmm/solver.py:495-520."""
    w = W.shape[1]
    U = st.U[(k, q)]
    r0 = U.shape[1]
    st.U[(k, q)] = np.concatenate([U, W], axis=1)
    d = st.tree.dim
    par = q >> d
    if (k - 1, par) in st.coff:
        at = st.coff[(k - 1, par)][q - (par << d)] + r0
        if (k - 1, par) in st.U:
            st.U[(k - 1, par)] = np.insert(st.U[(k - 1, par)], [at] * w, 0.0, axis=0)
        st.refresh_offsets(k - 1, par)


def _compress(F, tol):
    if tol == 0.0:
        L, R = tsvd(F, 0.0)
        return L, R, False
    return aca_block(F, tol)


def _squeeze_hybrid(st, k, p, q, tol, stats):
    """ifmm/solver.py:361-395."""
    F = st.blk["p2l"].get((k, p, q))
    if F is None:
        return
    A, B, bad = _compress(F, tol)
    if bad and not st.tree.sparse:  # sparse trees (extension): a full-rank ACA is exact and is absorbed
        stats.dense_kept += 1
        return
    stats.compressed += 1
    stats.max_rank = max(stats.max_rank, A.shape[1])
    stats.aca_ranks.append(A.shape[1])
    sc = np.sqrt(np.sum(A * A))
    W = _new_dirs(A, B, st.U[(k, q)], tol, sc)
    if W.shape[1]:
        _augment(st, k, q, W)
    dl = A @ (st.U[(k, q)].T @ B).T
    st.add("m2l", k, p, q, dl)
    st.add("m2l", k, q, p, dl.T.copy())
    st.drop_hybrid(k, p, q)


def _squeeze_near(st, k, p, q, tol, stats):
    """ifmm/solver.py:398-434."""
    F = st.blk["p2p"].get((k, p, q))
    if F is None:
        return
    A, B, bad = _compress(F, tol)
    if bad and not st.tree.sparse:  # sparse trees (extension): a full-rank ACA is exact and is absorbed
        stats.dense_kept += 1
        return
    stats.compressed += 1
    stats.max_rank = max(stats.max_rank, A.shape[1])
    stats.aca_ranks.append(A.shape[1])
    sc = np.sqrt(np.sum(A * A))
    W = _new_dirs(A, B, st.U[(k, q)], tol, sc)
    if W.shape[1]:
        _augment(st, k, q, W)
    W = _new_dirs(np.eye(B.shape[1]), A, st.U[(k, p)], tol, sc)
    if W.shape[1]:
        _augment(st, k, p, W)
    dl = (st.U[(k, p)].T @ A) @ (st.U[(k, q)].T @ B).T
    st.add("m2l", k, p, q, dl)
    st.add("m2l", k, q, p, dl.T.copy())
    st.drop_p2p(k, p, q)


def _eliminate(st: Blocks, k, i, tol, fac: Factor, stats: Stats, ils, dead):
    """One cluster elimination (ifmm/solver.py:195-311)."""
    U = st.U[(k, i)]
    n, r = U.shape
    if n + r == 0:  # an empty cluster of a sparse tree (extension): nothing to eliminate, no record
        dead[i] = True
        return
    S = np.zeros((n + r, n + r))
    S[:n, :n] = st.get("p2p", k, i, i)
    S[:n, n:] = U
    S[n:, :n] = U.T
    lu = lu_factor(S)
    rc = dgecon(lu[0], np.linalg.norm(S, 1), norm="1")[0]
    cond = 1.0 / max(rc, 1e-300) if np.isfinite(rc) else math.inf
    fac.max_cond[k] = max(fac.max_cond.get(k, 0.0), cond)
    if not np.isfinite(rc) or rc <= 1.0 / fac.cond_limit:
        if fac.on_singular != "record":
            raise SingularPivot(k, i, cond)
        fac.singular.append((k, i, cond))
    xp = sorted(j for j in st.pp.get((k, i), ()) if j != i and not dead[j])
    yp = sorted(st.plc.get((k, i), ()))
    cols = [("x", j, st.get("p2p", k, i, j)) for j in xp] + [("y", j, st.get("m2p", k, i, j)) for j in yp]
    wtot = sum(b.shape[1] for _, _, b in cols) + r
    C = np.zeros((n + r, wtot))
    sl, pos = [], 0
    for s, j, b in cols:
        C[:n, pos:pos + b.shape[1]] = b
        sl.append((s, j, slice(pos, pos + b.shape[1])))
        pos += b.shape[1]
    C[n:, pos:] = -np.eye(r)
    sl.append(("y", i, slice(pos, pos + r)))
    X = lu_solve(lu, C)
    rows = [("x", j, st.blk["p2p"][(k, j, i)]) for j in xp] + [("z", j, st.blk["p2l"][(k, j, i)]) for j in yp]
    fpp, fhy = set(), set()

    def scatter(rs, rj, Y):
        for cs, l, s in sl:
            dl = -Y[:, s]
            if rs == "x" and cs == "x":
                st.add("p2p", k, rj, l, dl)
                if rj != l:
                    fpp.add((min(rj, l), max(rj, l)))
            elif rs == "x":
                st.add("m2p", k, rj, l, dl)
                if rj != l:
                    fhy.add((l, rj))
            elif cs == "x":
                st.add("p2l", k, rj, l, dl)
                if rj != l:
                    fhy.add((rj, l))
            else:
                st.add("m2l", k, rj, l, dl)

    for rs, j, b in rows:
        scatter(rs, j, b @ X[:n])
    scatter("z", i, -X[n:])
    dead[i] = True
    fac.recs.append(Rec(k, i, lu, n, r, xp, yp))
    for p, q in sorted(fhy):
        if q in ils[p]:
            _squeeze_hybrid(st, k, p, q, tol, stats)
    for p, q in sorted(fpp):
        if q in ils[p]:
            _squeeze_near(st, k, p, q, tol, stats)


def _consolidate(st: Blocks, k, batch, rank_tol, fac: Factor):
    """Rank-growth control -- NOT reference behaviour: a working
    restatement of what the reference's unused `_maybe_consolidate`
    (ifmm/solver.py:437-492) is after, and the checker of the GPU extension
    `factorize(..., rank_tol=)` (csrc/consolidate.cu).

    Right before the clusters of `batch` are eliminated, each one's coupling row
    Rw = [M2L(i, l) for every partner l | its rows of the parent's basis] is
    truncated by a column-pivoted QR of Rw^T at |R_jj| > rank_tol |R_00|, T_i = an
    orthonormal basis of the kept left factor, and U_i <- U_i T_i,
    M2L(i, l) <- T_i^T M2L(i, l) T_l (T_l = I for clusters outside the batch),
    parent rows <- T_i^T rows.  Every T of a batch is computed from the blocks as
    they were before the batch's rotations (the GPU runs them concurrently)."""
    tree, d = st.tree, st.tree.dim
    part = {}
    inb = set(int(i) for i in batch)
    for (kk, i, j) in st.blk["m2l"]:
        if kk == k and i in inb and j != i:
            part.setdefault(i, []).append(j)
    T = {}
    old_r = {}
    for i in sorted(inb):
        r = st.r(k, i)
        if r == 0 or (k, i, i) in st.blk["m2l"]:
            continue
        blocks = [st.get("m2l", k, i, l) for l in sorted(part.get(i, [])) if st.r(k, l) > 0]
        par = i >> d
        if k > 2:
            st.refresh_offsets(k - 1, par)
            o = st.coff[(k - 1, par)]
            c = i - (par << d)
            blocks.append(st.U[(k - 1, par)][o[c]:o[c + 1], :])
        if not blocks:
            continue
        Rw = np.concatenate(blocks, axis=1)
        if Rw.shape[1] == 0:
            continue
        _, R, P = qr(Rw.T, mode="economic", pivoting=True)
        dg = np.abs(np.diag(R))
        rc = int(np.sum(dg > rank_tol * dg[0])) if dg[0] > 0 else r
        rc = max(rc, 1)
        fac.rank_control[0] += r
        fac.rank_control[1] += min(rc, r)
        if rc >= r:
            continue
        Lm = np.zeros((r, rc))
        Lm[P, :] = R[:rc, :].T
        T[i] = qr(Lm, mode="economic")[0]
        old_r[i] = r
    if not T:
        return
    # pad helpers: blocks are lazily sized; bring them to the pre-rotation ranks first
    blocks_new = {}
    for i, Ti in T.items():
        for l in part.get(i, []):
            B = st.get("m2l", k, i, l)
            Tl = T.get(l)
            blocks_new[(k, i, l)] = Ti.T @ B @ Tl if Tl is not None else Ti.T @ B
            if l not in T:
                blocks_new[(k, l, i)] = st.get("m2l", k, l, i) @ Ti
    prow = {}
    if k > 2:
        for i, Ti in T.items():
            par = i >> d
            o = st.coff[(k - 1, par)]
            c = i - (par << d)
            prow[i] = Ti.T @ st.U[(k - 1, par)][o[c]:o[c + 1], :]
    for key, B in blocks_new.items():
        st.blk["m2l"][key] = B
    for i, Ti in T.items():
        st.U[(k, i)] = st.U[(k, i)] @ Ti
    if k > 2:
        for par in sorted(set(i >> d for i in T)):
            o = st.coff[(k - 1, par)]
            P0 = st.U[(k - 1, par)]
            rows = []
            for c in range(1 << d):
                ch = (par << d) + c
                rows.append(prow[ch] if ch in prow else P0[o[c]:o[c + 1], :])
            st.U[(k - 1, par)] = np.concatenate(rows, axis=0)
            st.refresh_offsets(k - 1, par)


def _top(fac: Factor):
    """Dense LU of the level-2 M2L system (ifmm/solver.py:528-546)."""
    st, tree = fac.st, fac.tree
    nc = tree.n_clusters(2)
    dims = np.array([st.r(2, i) for i in range(nc)])
    off = np.concatenate([[0], np.cumsum(dims)]).astype(int)
    T = np.zeros((off[-1], off[-1]))
    for i in range(nc):
        for j in range(nc):
            b = st.blk["m2l"].get((2, i, j))
            if b is not None:
                T[off[i]:off[i] + b.shape[0], off[j]:off[j] + b.shape[1]] = b
    fac.top_lu = lu_factor(T)
    fac.top_off = off


def factorize(st: Blocks, tol=None, order="morton", release_m2l=True, cond_limit=COND_LIMIT,
              on_singular="raise", progress=None, rank_tol=None) -> Factor:
    """ifmm/solver.py:106-153 with a selectable intra-level order.  `on_singular="record"`
    keeps going past a pivot the reference would reject (ifmm/solver.py:214-218) and lists it
    in `fac.singular`; `progress(k, fac)` is called after each level."""
    tree = st.tree
    tol = st.tol if tol is None else tol
    fac = Factor(st, tree, tol, order=order, cond_limit=cond_limit, on_singular=on_singular)
    fac.r_m = st.max_init_rank
    K = tree.depth
    for k in range(K, 1, -1):
        if k < K:
            _parent_near(st, k)
            if release_m2l:
                for key in [kk for kk in st.blk["m2l"] if kk[0] == k + 1]:
                    del st.blk["m2l"][key]
        stats = Stats(clusters=tree.n_clusters(k))
        fac.stats[k] = stats
        ils = [set(x) for x in tree.ilist[k]]
        dead = np.zeros(tree.n_clusters(k), dtype=bool)
        for batch in elimination_order(tree, k, order):
            # rank_tol: extension, see _consolidate (off in the reference algorithm)
            if rank_tol is not None and order != "morton":
                _consolidate(st, k, batch, rank_tol, fac)
            for i in batch:
                if rank_tol is not None and order == "morton":
                    _consolidate(st, k, [i], rank_tol, fac)
                _eliminate(st, k, int(i), tol, fac, stats, ils, dead)
        fac.r_m = max(fac.r_m, stats.max_rank)
        if progress is not None:
            progress(k, fac)
    _top(fac)
    if release_m2l:
        for key in [kk for kk in st.blk["m2l"] if kk[0] == 2]:
            del st.blk["m2l"][key]
    return fac


def solve(fac: Factor, rhs):
    """Forward replay, top solve, reverse back-substitution (ifmm/solver.py:549-626).
    Accepts (N,) or (N, nrhs)."""
    st, tree = fac.st, fac.tree
    rhs = np.asarray(rhs, dtype=float)
    one = rhs.ndim == 1
    B = rhs.reshape(len(tree.points), -1)[tree.perm]
    K, d = tree.depth, tree.dim
    nr = B.shape[1]
    bx = {(K, i): B[tree.leaf_off[i]:tree.leaf_off[i + 1]].copy() for i in range(tree.n_clusters(K))}
    bz = {}
    gs = []
    cur = K
    for rec in fac.recs:
        k, i = rec.level, rec.index
        if k != cur:
            for c in range(tree.n_clusters(k)):
                bx[(k, c)] = np.concatenate([bz.get((k + 1, ch), np.zeros((0, nr)))
                                             for ch in range(c << d, (c + 1) << d)])
            cur = k
        g = lu_solve(rec.lu, np.concatenate([bx[(k, i)], np.zeros((rec.r, nr))]))
        gs.append(g)
        for j in rec.xp:
            bx[(k, j)] -= st.blk["p2p"][(k, j, i)] @ g[:rec.n]
        for j in rec.yp:
            bz[(k, j)] -= st.blk["p2l"][(k, j, i)] @ g[:rec.n]
        bz[(k, i)] = g[rec.n:].copy()
    off = fac.top_off
    yt = lu_solve(fac.top_lu, np.concatenate([bz.get((2, c), np.zeros((0, nr))) for c in range(tree.n_clusters(2))]))
    y = {(2, c): yt[off[c]:off[c + 1]] for c in range(tree.n_clusters(2))}
    xv = {}
    by = {}
    for idx, rec in enumerate(fac.recs):
        by.setdefault(rec.level, []).append((rec, gs[idx]))
    for k in range(2, K + 1):
        for rec, g in reversed(by[k]):
            i = rec.index
            top = np.zeros((rec.n, nr))
            for j in rec.xp:
                if (k, j) in xv:  # (an empty cluster of a sparse tree has no unknowns)
                    top += st.blk["p2p"][(k, i, j)] @ xv[(k, j)]
            for j in rec.yp:
                top += st.blk["m2p"][(k, i, j)] @ y[(k, j)]
            sol = g - lu_solve(rec.lu, np.concatenate([top, -y[(k, i)]]))
            xv[(k, i)] = sol[:rec.n]
            if k < K:
                o = st.coff[(k, i)]
                for c, ch in enumerate(range(i << d, (i + 1) << d)):
                    y[(k + 1, ch)] = sol[o[c]:o[c + 1]]
    out = np.empty((len(tree.points), nr))
    for i in range(tree.n_clusters(K)):
        if (K, i) in xv:
            out[tree.leaf_off[i]:tree.leaf_off[i + 1]] = xv[(K, i)]
    res = np.empty_like(out)
    res[tree.perm] = out
    return res[:, 0] if one else res


# --------------------------------------------------------------------------
# BASELINE.json configurations (SURVEY.md section 8c adapter)
# --------------------------------------------------------------------------
CONFIGS = {
    # name: (N, kernel, depth, p, tol, rhs kind)
    "C1": (4096, "inv_r", 3, 4, 1e-8, "manufactured"),
    "C2": (65536, "log_r", 5, 5, 1e-6, "normal"),
    "C3": (1048576, "inv_r", 7, 4, 1e-6, "normal"),
    "C5": (16777216, "log_r", 9, 4, 1e-6, "normal32"),
}


def baseline_kernel(name, n):
    """Adapter: x' = 2x-1 maps [0,1]^2 to the reference box; the system is divided by
    sqrt(N) so the diagonal sqrt(N) becomes 1 and K(x,y)=1/|x-y| becomes (2/r')/sqrt(N),
    log|x-y| becomes (ln r' - ln 2)/sqrt(N)."""
    s = 1.0 / math.sqrt(n)
    if name == "inv_r":
        return KernelSpec("inv_r", scale=2.0 * s)
    if name == "log_r":
        return KernelSpec("log_r", scale=s, shift=-math.log(2.0))
    raise ValueError(name)


def baseline_points(n, seed=0):
    """Seeded points uniform in [0,1]^2, mapped to [-1,1]^2 (seed 0)."""
    rng = np.random.default_rng(seed)
    return 2.0 * rng.random((n, 2)) - 1.0


def baseline_rhs(n, kind, seed=0):
    rng = np.random.default_rng([seed, 1])
    if kind == "normal32":
        return rng.standard_normal((n, 32))
    return rng.standard_normal(n) if kind == "normal" else rng.uniform(-1.0, 1.0, n)
