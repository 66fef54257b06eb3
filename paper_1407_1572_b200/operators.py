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
