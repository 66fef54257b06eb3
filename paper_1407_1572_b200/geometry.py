"""Point sets and the uniform 2^d cluster tree (mirror of ifmm/geometry.py).

The tree is built on the GPU by libifmm_b200 (Morton codes, stable radix sort,
leaf offsets, duplicate scan); neighbour / interaction lists and the 3^d
elimination colouring come back as integer arrays.  `Cluster` objects are
materialised lazily for API compatibility with the reference.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib

BOX_HALF_WIDTH = 1.0      # ifmm/geometry.py:30
DUPLICATE_TOL = 1e-14     # ifmm/geometry.py:31


@dataclass
class PointSet:
    """Points in the reference box [-1, 1]^dim (ifmm/geometry.py:34-65).

    Shape and box are checked here; duplicate points (distance <= 1e-14) are
    rejected by the GPU tree build with the reference's message."""

    dim: int
    points: np.ndarray

    def __post_init__(self):
        self.points = np.ascontiguousarray(self.points, dtype=float)
        if self.dim not in (1, 2, 3):
            raise ValueError(f"dim must be 1, 2 or 3, got {self.dim}")
        if self.points.ndim != 2 or self.points.shape[1] != self.dim:
            raise ValueError(f"points must have shape (n, {self.dim}), got {self.points.shape}")
        if np.abs(self.points).max(initial=0.0) > BOX_HALF_WIDTH:
            raise ValueError("point outside the reference box [-1, 1]^d")

    def __len__(self) -> int:
        return len(self.points)


@dataclass
class Cluster:
    level: int
    index: int
    grid: tuple
    center: np.ndarray
    half_width: float
    children: list = field(default_factory=list)
    point_range: tuple | None = None
    neighbors: list = field(default_factory=list)
    interaction_list: list = field(default_factory=list)
    eliminated: bool = False


def morton_encode(grid: np.ndarray, dim: int, bits: int) -> np.ndarray:
    """x bit least significant (ifmm/geometry.py:124-131)."""
    grid = np.asarray(grid, dtype=np.int64)
    codes = np.zeros(grid.shape[0], dtype=np.int64)
    for b in range(bits):
        for ax in range(dim):
            codes |= ((grid[:, ax] >> b) & 1) << (b * dim + ax)
    return codes


def morton_decode(codes: np.ndarray, dim: int, bits: int) -> np.ndarray:
    codes = np.asarray(codes, dtype=np.int64)
    grid = np.zeros((codes.shape[0], dim), dtype=np.int64)
    for b in range(bits):
        for ax in range(dim):
            grid[:, ax] |= ((codes >> (b * dim + ax)) & 1) << b
    return grid


class ClusterTree:
    """Uniform 2^d tree over Morton-permuted points (ifmm/geometry.py:88-121).

    Owns the device-side tree handle."""

    def __init__(self, handle, ps: PointSet, depth: int):
        self._h = handle
        self.depth = depth
        self.dim = ps.dim
        n = len(ps)
        perm = np.empty(n, dtype=np.int64)
        _lib.check(_lib.lib.ifmm_tree_permutation(self._h, _lib.ptr(perm)))
        off = np.empty((1 << (self.dim * depth)) + 1, dtype=np.int64)
        _lib.check(_lib.lib.ifmm_tree_leaf_offsets(self._h, _lib.ptr(off)))
        self.point_permutation = perm
        self.leaf_offsets = off
        self.points = ps.points[perm]
        self._levels = None
        self._lists = {}

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            _lib.lib.ifmm_tree_free(h)

    @property
    def handle(self):
        return self._h

    @property
    def n_points(self) -> int:
        return len(self.points)

    def lists(self, level: int):
        """(nbr_off, nbr, il_off, il) CSR arrays of `level`."""
        if level not in self._lists:
            sizes = np.zeros(2, dtype=np.int64)
            _lib.check(_lib.lib.ifmm_tree_lists(self._h, level, None, None, None, None, _lib.ptr(sizes)))
            nc = 1 << (self.dim * level)
            nbo = np.empty(nc + 1, dtype=np.int32)
            nb = np.empty(max(1, sizes[0]), dtype=np.int32)
            ilo = np.empty(nc + 1, dtype=np.int32)
            il = np.empty(max(1, sizes[1]), dtype=np.int32)
            _lib.check(_lib.lib.ifmm_tree_lists(self._h, level, _lib.ptr(nbo), _lib.ptr(nb), _lib.ptr(ilo),
                                                _lib.ptr(il), _lib.ptr(sizes)))
            self._lists[level] = (nbo, nb[:sizes[0]], ilo, il[:sizes[1]])
        return self._lists[level]

    def colours(self, level: int) -> np.ndarray:
        out = np.empty(1 << (self.dim * level), dtype=np.int32)
        _lib.check(_lib.lib.ifmm_tree_colours(self._h, level, _lib.ptr(out)))
        return out

    @property
    def levels(self) -> dict:
        if self._levels is None:
            self._levels = {k: self._make_level(k) for k in range(1, self.depth + 1)}
        return self._levels

    def _make_level(self, k: int) -> list:
        nbo, nb, ilo, il = self.lists(k)
        nk = 1 << (self.dim * k)
        grid = morton_decode(np.arange(nk), self.dim, k)
        w = 2.0 * BOX_HALF_WIDTH / (2 ** k)
        centers = -BOX_HALF_WIDTH + (grid + 0.5) * w
        out = []
        for i in range(nk):
            c = Cluster(level=k, index=i, grid=tuple(int(g) for g in grid[i]), center=centers[i], half_width=w / 2)
            if k < self.depth:
                c.children = list(range((1 << self.dim) * i, (1 << self.dim) * (i + 1)))
            else:
                c.point_range = (int(self.leaf_offsets[i]), int(self.leaf_offsets[i + 1]))
            c.neighbors = [int(v) for v in nb[nbo[i]:nbo[i + 1]]]
            c.interaction_list = [int(v) for v in il[ilo[i]:ilo[i + 1]]]
            out.append(c)
        return out

    def clusters(self, level: int) -> list:
        return self.levels[level]

    def leaf_points(self, index: int) -> np.ndarray:
        return self.points[self.leaf_offsets[index]:self.leaf_offsets[index + 1]]

    def cluster_point_range(self, level: int, index: int) -> tuple:
        step = 1 << (self.dim * (self.depth - level))
        return int(self.leaf_offsets[index * step]), int(self.leaf_offsets[(index + 1) * step])


def build_tree(ps: PointSet, depth: int, allow_empty_leaves: bool = False) -> ClusterTree:
    """GPU tree build (ifmm/geometry.py:174-226); raises ValueError like the
    reference for depth < 2, duplicate points and empty leaves.

    allow_empty_leaves (extension, for clustered inputs such as BASELINE config
    4's Gaussian mixture): leaf cells without points are accepted; their
    clusters carry no unknowns."""
    if not isinstance(ps, PointSet):
        raise TypeError("build_tree expects a PointSet")
    h = ctypes.c_void_p()
    fn = _lib.lib.ifmm_tree_build_sparse if allow_empty_leaves else _lib.lib.ifmm_tree_build
    _lib.check(fn(_lib.ptr(ps.points), len(ps), ps.dim, int(depth), _lib.PTR_HOST, ctypes.byref(h)))
    return ClusterTree(h, ps, int(depth))


def compute_lists(tree: ClusterTree) -> ClusterTree:
    """Lists are computed with the tree (ifmm/geometry.py:229-262); kept for API parity."""
    return tree
