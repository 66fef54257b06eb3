"""Operator store on the GPU (mirror of ifmm/operators.py).

`init_operators` assembles the leaf near field, the Chebyshev bases and the
M2L operators in HBM (libifmm_b200 store_init); `fmm_matvec` applies the
compressed operator with device kernels.  Block accessors download on demand
for inspection and tests.
"""
from __future__ import annotations

import ctypes
import weakref

import numpy as np

from . import _lib
from .geometry import ClusterTree
from .kernels import Kernel


class _BasisView:
    def __init__(self, store):
        # weak: the store owns its views; a strong back-reference would be a cycle that keeps
        # the store's HBM alive until the garbage collector runs
        self._s = weakref.proxy(store)

    def __getitem__(self, key):
        k, i = key
        n, r = self._s.part_dim(k, i), self._s.rank(k, i)
        out = np.empty((r, n))  # column-major n x r
        _lib.check(_lib.lib.ifmm_store_basis(self._s.handle, k, i, _lib.ptr(out)))
        return out.T.copy()


class _M2LView:
    def __init__(self, store):
        # weak: the store owns its views; a strong back-reference would be a cycle that keeps
        # the store's HBM alive until the garbage collector runs
        self._s = weakref.proxy(store)

    def __getitem__(self, key):
        k, i, j = key
        ri, rj = self._s.rank(k, i), self._s.rank(k, j)
        out = np.empty((rj, ri))
        _lib.check(_lib.lib.ifmm_store_m2l(self._s.handle, k, i, j, _lib.ptr(out)))
        return out.T.copy()


class _P2PView:
    def __init__(self, store):
        # weak: the store owns its views; a strong back-reference would be a cycle that keeps
        # the store's HBM alive until the garbage collector runs
        self._s = weakref.proxy(store)

    def __getitem__(self, key):
        k, i, j = key
        if k != self._s.tree.depth:
            raise KeyError(key)  # the initial store holds leaf near fields only
        ni, nj = self._s.part_dim(k, i), self._s.part_dim(k, j)
        out = np.empty((nj, ni))
        _lib.check(_lib.lib.ifmm_store_p2p(self._s.handle, i, j, _lib.ptr(out)))
        return out.T.copy()


class OperatorStore:
    """Initial extended system resident in HBM (ifmm/operators.py:42-137)."""

    def __init__(self, handle, tree: ClusterTree, kernel: Kernel, p: int, tol: float):
        self._h = handle
        self.tree = tree
        self.kernel = kernel
        self.p = p
        self.tol = tol
        self._dims = {}
        r = ctypes.c_int()
        _lib.check(_lib.lib.ifmm_store_max_init_rank(self._h, ctypes.byref(r)))
        self.max_init_rank = r.value
        self.l2p = _BasisView(self)
        self.m2l = _M2LView(self)
        self.p2p = _P2PView(self)

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            _lib.lib.ifmm_store_free(h)

    @property
    def handle(self):
        return self._h

    def _level_dims(self, k):
        if k not in self._dims:
            nc = 1 << (self.tree.dim * k)
            n = np.empty(nc, dtype=np.int32)
            r = np.empty(nc, dtype=np.int32)
            _lib.check(_lib.lib.ifmm_store_dims(self._h, k, _lib.ptr(n), _lib.ptr(r)))
            self._dims[k] = (n, r)
        return self._dims[k]

    def rank(self, k: int, i: int) -> int:
        return int(self._level_dims(k)[1][i])

    def part_dim(self, k: int, i: int) -> int:
        return int(self._level_dims(k)[0][i])

    @property
    def nbytes(self) -> dict:
        """Bytes of the assembled operators as stored (leaf P2P once per pair,
        M2L both orientations, bases): assembly writes them, matvec reads them."""
        out = np.zeros(3)
        _lib.check(_lib.lib.ifmm_store_bytes(self._h, _lib.ptr(out)))
        return {"p2p": out[0], "m2l": out[1], "basis": out[2]}

    def ranks(self, k: int) -> np.ndarray:
        return self._level_dims(k)[1].copy()

    def child_slices(self, k: int, i: int) -> list:
        """Row slices of the children's multipoles in the basis of non-leaf
        cluster (k, i) (ifmm/operators.py:130-137)."""
        nch = 1 << self.tree.dim
        out, lo = [], 0
        for c in range(nch * i, nch * (i + 1)):
            r = self.rank(k + 1, c)
            out.append(slice(lo, lo + r))
            lo += r
        return out


def init_operators(tree: ClusterTree, kernel: Kernel, p: int = 8, tol: float = 1e-14) -> OperatorStore:
    """Build the initial operator set on the GPU (ifmm/operators.py:164-177)."""
    if not isinstance(kernel, Kernel):
        raise ValueError("kernel must be a paper_1407_1572_b200.Kernel (Python callables cannot run on the GPU)")
    probes = _lib.aca_probe_table()
    h = ctypes.c_void_p()
    _lib.check(_lib.lib.ifmm_store_init(tree.handle, kernel.kernel_id, float(kernel.a), float(kernel.scale),
                                        float(kernel.shift), int(p), float(tol), _lib.ptr(probes),
                                        probes.shape[0] - 1, ctypes.byref(h)))
    return OperatorStore(h, tree, kernel, int(p), float(tol))


def load_operator_blocks(store: OperatorStore, bases: dict, m2l: dict, p2p: dict) -> OperatorStore:
    """Test hook: overwrite the GPU store's initial operators with
    blocks built elsewhere, e.g. a reference OperatorStore's `l2p`, `m2l`, `p2p`
    dicts (ifmm/operators.py:42-137), so factorize runs on bit-identical inputs.
    bases[(k, i)] n x r; m2l[(k, i, j)] r_i x r_j on interaction-list pairs;
    p2p[(k, i, j)] n_i x n_j on leaf neighbour pairs.  Shapes must match the
    store's (same tree, same initial ranks); ValueError otherwise."""
    K = store.tree.depth

    def col(a):
        return np.asfortranarray(np.asarray(a, dtype=float))

    for (k, i), U in bases.items():
        if U.shape != (store.part_dim(k, i), store.rank(k, i)):
            raise ValueError(f"basis ({k}, {i}) has shape {U.shape}, the store {store.part_dim(k, i), store.rank(k, i)}")
        _lib.check(_lib.lib.ifmm_store_set_basis(store.handle, k, i, _lib.ptr(col(U))))
    for (k, i, j), M in m2l.items():
        if M.shape != (store.rank(k, i), store.rank(k, j)):
            raise ValueError(f"M2L ({k}, {i}, {j}) has shape {M.shape}")
        _lib.check(_lib.lib.ifmm_store_set_m2l(store.handle, k, i, j, _lib.ptr(col(M))))
    for (k, i, j), P in p2p.items():
        if k != K:
            continue  # the initial store holds the leaf near field only
        _lib.check(_lib.lib.ifmm_store_set_p2p(store.handle, i, j, _lib.ptr(col(P))))
    return store


def fmm_matvec(store: OperatorStore, tree: ClusterTree, charges):
    """Apply the compressed operator (ifmm/operators.py:282-330).  `charges` is
    (N,) or (N, nrhs), numpy or torch (CUDA tensors stay on the device)."""
    n = tree.n_points
    p_in, kind, nr, keep, is_torch, one_d = _lib.as_input(charges, n)
    out, p_out = _lib.alloc_output(keep, kind, n, nr, one_d)
    _lib.check(_lib.lib.ifmm_matvec(store.handle, p_in, p_out, nr, kind))
    if is_torch and kind == _lib.PTR_HOST:
        import torch
        out = torch.from_numpy(out)
    return out[:, 0] if one_d else out


# ----------------------------------------------------------------------
# extended sparse system: verification / export path (ifmm/operators.py:333-486).
# The slot table and the matrix come from the library (csrc/extended.cu: a
# device scatter of the store's blocks); rhs / solution maps are index arrays.
# ----------------------------------------------------------------------

_SYMS = "xyz"


def _slot_table(store: OperatorStore):
    cnt = ctypes.c_int64()
    _lib.check(_lib.lib.ifmm_extended_layout(store.handle, ctypes.byref(cnt), None, None, None, None))
    cols = [np.zeros(cnt.value, dtype=np.int32) for _ in range(4)]
    _lib.check(_lib.lib.ifmm_extended_layout(store.handle, ctypes.byref(cnt), *[_lib.ptr(c) for c in cols]))
    return cols


def extended_layout(store: OperatorStore, tree: ClusterTree) -> list:
    """Unknown slots of the extended system as (symbol, level, cluster, dim), in
    the reference's order (ifmm/operators.py:338-364): leaf (x, z) pairs in
    Morton order, then per coarser level each cluster's children's y slots and
    its own z slot (none at level 1)."""
    sym, lev, idx, dim = _slot_table(store)
    return [(_SYMS[a], int(b), int(c), int(d)) for a, b, c, d in zip(sym, lev, idx, dim)]


def assemble_extended_dense(store: OperatorStore, tree: ClusterTree, cap: int = 4096):
    """The initial extended system as a dense matrix (ifmm/operators.py:367-445),
    scattered from the device store.  Returns (matrix, slots); ValueError above
    `cap` unknowns."""
    m = ctypes.c_int64()
    _lib.check(_lib.lib.ifmm_extended_dense(store.handle, int(cap), ctypes.byref(m), None))
    buf = np.empty((m.value, m.value))
    _lib.check(_lib.lib.ifmm_extended_dense(store.handle, int(cap), ctypes.byref(m), _lib.ptr(buf)))
    return np.ascontiguousarray(buf.T), extended_layout(store, tree)  # the library writes column-major


def _x_positions(store: OperatorStore, tree: ClusterTree) -> np.ndarray:
    """Extended position of every point, in Morton (permuted) order."""
    sym, _, idx, dim = _slot_table(store)
    start = np.concatenate([[0], np.cumsum(dim.astype(np.int64))[:-1]])
    xs = sym == 0
    ox = np.empty(int(xs.sum()), dtype=np.int64)
    ox[idx[xs]] = start[xs]                      # x slot offset of every leaf
    off = np.asarray(tree.leaf_offsets, dtype=np.int64)
    leaf = np.repeat(np.arange(len(off) - 1), np.diff(off))
    return ox[leaf] + (np.arange(off[-1]) - off[leaf])


def extended_rhs(store: OperatorStore, tree: ClusterTree, b) -> np.ndarray:
    """Extended right-hand side: b on the particle slots, zeros elsewhere
    (ifmm/operators.py:448-459)."""
    _, _, _, dim = _slot_table(store)
    out = np.zeros(int(dim.astype(np.int64).sum()))
    out[_x_positions(store, tree)] = np.asarray(b, dtype=float)[tree.point_permutation]
    return out


def extended_restrict_x(store: OperatorStore, tree: ClusterTree, xe) -> np.ndarray:
    """The original unknowns of an extended solution, in original point order
    (ifmm/operators.py:462-477)."""
    res = np.empty(tree.n_points)
    res[tree.point_permutation] = np.asarray(xe)[_x_positions(store, tree)]
    return res


def dump_extended(store: OperatorStore, tree: ClusterTree, path, cap: int = 4096) -> None:
    """Nonzeros of the extended matrix as 'row col value' lines after a header
    line -- the reference's text format (ifmm/operators.py:480-486)."""
    A, _ = assemble_extended_dense(store, tree, cap=cap)
    rows, cols = np.nonzero(A)
    with open(path, "w") as fh:
        fh.write(f"# extended system, dimension {A.shape[0]}\n")
        fh.writelines(f"{r} {c} {v:.17g}\n" for r, c, v in zip(rows, cols, A[rows, cols]))
