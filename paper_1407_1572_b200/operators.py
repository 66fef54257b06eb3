"""Operator store on the GPU (mirror of ifmm/operators.py).

`init_operators` assembles the leaf near field, the Chebyshev bases and the
M2L operators in HBM (libifmm_b200 store_init); `fmm_matvec` applies the
compressed operator with device kernels.  Block accessors download on demand
for inspection and tests.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .geometry import ClusterTree
from .kernels import Kernel


class _BasisView:
    def __init__(self, store):
        self._s = store

    def __getitem__(self, key):
        k, i = key
        n, r = self._s.part_dim(k, i), self._s.rank(k, i)
        out = np.empty((r, n))  # column-major n x r
        _lib.check(_lib.lib.ifmm_store_basis(self._s.handle, k, i, _lib.ptr(out)))
        return out.T.copy()


class _M2LView:
    def __init__(self, store):
        self._s = store

    def __getitem__(self, key):
        k, i, j = key
        ri, rj = self._s.rank(k, i), self._s.rank(k, j)
        out = np.empty((rj, ri))
        _lib.check(_lib.lib.ifmm_store_m2l(self._s.handle, k, i, j, _lib.ptr(out)))
        return out.T.copy()


class _P2PView:
    def __init__(self, store):
        self._s = store

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
# extended sparse system: verification / export path (ifmm/operators.py:333-486)
# ----------------------------------------------------------------------


def extended_layout(store: OperatorStore, tree: ClusterTree) -> list:
    """Slot order of the extended system's unknowns (ifmm/operators.py:338-364):
    leaf (x_i, z_i) pairs in Morton order, then per coarser level each
    cluster's children's y slots followed by its own z slot (none at level 1)."""
    kappa = tree.depth
    nch = 1 << tree.dim
    slots = []
    off = tree.leaf_offsets
    for i in range(1 << (tree.dim * kappa)):
        slots.append(("x", kappa, i, int(off[i + 1] - off[i])))
        slots.append(("z", kappa, i, store.rank(kappa, i)))
    for k in range(kappa - 1, 0, -1):
        for i in range(1 << (tree.dim * k)):
            for ch in range(nch * i, nch * (i + 1)):
                slots.append(("y", k + 1, ch, store.rank(k + 1, ch)))
            if k >= 2:
                slots.append(("z", k, i, store.rank(k, i)))
    return slots


def assemble_extended_dense(store: OperatorStore, tree: ClusterTree, cap: int = 4096):
    """Materialise the initial extended system densely on the host
    (ifmm/operators.py:367-445): particle equations, charge-lumping equations
    and local-definition equations, blocks downloaded from the device store.
    Returns (matrix, slots).  Raises ValueError above `cap` unknowns."""
    slots = extended_layout(store, tree)
    offsets, pos = {}, 0
    for sym, k, i, dim in slots:
        offsets[(sym, k, i)] = pos
        pos += dim
    m = pos
    if m > cap:
        raise ValueError(f"extended dimension {m} exceeds cap {cap}")
    A = np.zeros((m, m))
    kappa, nch = tree.depth, 1 << tree.dim
    leaves = tree.levels[kappa]

    def xcols(k, i):
        if k == kappa:
            return [(offsets[("x", k, i)], store.part_dim(k, i))]
        return [(offsets[("y", k + 1, ch)], store.rank(k + 1, ch)) for ch in range(nch * i, nch * (i + 1))]

    for c in leaves:  # leaf particle equations
        i = c.index
        r0, n_i = offsets[("x", kappa, i)], store.part_dim(kappa, i)
        for j in c.neighbors:
            blk = store.p2p[(kappa, i, j)]
            c0 = offsets[("x", kappa, j)]
            A[r0:r0 + n_i, c0:c0 + blk.shape[1]] = blk
        U = store.l2p[(kappa, i)]
        z0 = offsets[("z", kappa, i)]
        A[r0:r0 + n_i, z0:z0 + U.shape[1]] = U
    for k in range(kappa, 1, -1):  # charge-lumping equations
        for i in range(1 << (tree.dim * k)):
            U = store.l2p[(k, i)]
            r0, r_i = offsets[("z", k, i)], U.shape[1]
            col = 0
            for c0, w in xcols(k, i):
                A[r0:r0 + r_i, c0:c0 + w] = U[col:col + w, :].T
                col += w
            y0 = offsets[("y", k, i)]
            A[r0:r0 + r_i, y0:y0 + r_i] -= np.eye(r_i)
    for k in range(2, kappa + 1):  # local-definition equations
        for c in tree.levels[k]:
            i = c.index
            r0, r_i = offsets[("y", k, i)], store.rank(k, i)
            z0 = offsets[("z", k, i)]
            A[r0:r0 + r_i, z0:z0 + r_i] -= np.eye(r_i)
            for j in c.interaction_list:
                blk = store.m2l[(k, i, j)]
                y0 = offsets[("y", k, j)]
                A[r0:r0 + r_i, y0:y0 + blk.shape[1]] = blk
            if k > 2:
                pk, pi = k - 1, i // nch
                Upar = store.l2p[(pk, pi)][store.child_slices(pk, pi)[i % nch], :]
                zp = offsets[("z", pk, pi)]
                A[r0:r0 + r_i, zp:zp + Upar.shape[1]] = Upar
    return A, slots


def extended_rhs(store: OperatorStore, tree: ClusterTree, b) -> np.ndarray:
    """Extended right-hand side: b (Morton order) on the x slots, 0 elsewhere
    (ifmm/operators.py:448-459)."""
    slots = extended_layout(store, tree)
    b_m = np.asarray(b, dtype=float)[tree.point_permutation]
    out = np.zeros(sum(s[3] for s in slots))
    pos = 0
    for sym, k, i, dim in slots:
        if sym == "x":
            lo, hi = int(tree.leaf_offsets[i]), int(tree.leaf_offsets[i + 1])
            out[pos:pos + dim] = b_m[lo:hi]
        pos += dim
    return out


def extended_restrict_x(store: OperatorStore, tree: ClusterTree, xe) -> np.ndarray:
    """Original unknowns (original point order) of an extended solution
    (ifmm/operators.py:462-477)."""
    slots = extended_layout(store, tree)
    out = np.empty(tree.n_points)
    pos = 0
    for sym, k, i, dim in slots:
        if sym == "x":
            lo, hi = int(tree.leaf_offsets[i]), int(tree.leaf_offsets[i + 1])
            out[lo:hi] = xe[pos:pos + dim]
        pos += dim
    res = np.empty_like(out)
    res[tree.point_permutation] = out
    return res


def dump_extended(store: OperatorStore, tree: ClusterTree, path, cap: int = 4096) -> None:
    """Write the extended matrix as 'row col value' nonzero triplets with a
    one-line header (ifmm/operators.py:480-486, same format)."""
    A, _ = assemble_extended_dense(store, tree, cap=cap)
    rows, cols = np.nonzero(A)
    with open(path, "w") as fh:
        fh.write(f"# extended system, dimension {A.shape[0]}\n")
        for r, c in zip(rows, cols):
            fh.write(f"{r} {c} {A[r, c]:.17g}\n")
