"""GPU factorization and solve (mirror of ifmm/solver.py).

`factorize` runs the whole level-by-level, colour-batched elimination in
libifmm_b200 (csrc/factor.cu); `solve` replays it for one or many right-hand
sides (csrc/solve.cu).  Exceptions follow the reference: SingularPivotError
for numerically singular pivots, ValueError for bad shapes.
"""
from __future__ import annotations

import ctypes
import logging
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import SingularPivotError
from .geometry import ClusterTree
from .operators import OperatorStore

logger = logging.getLogger("ifmm")

PIVOT_CONDITION_LIMIT = 1e12  # ifmm/solver.py:50

__all__ = ["IfmmFactorization", "LevelStats", "SingularPivotError", "factorize", "solve"]


@dataclass
class LevelStats:
    clusters: int = 0
    max_rank: int = 0
    fillins_compressed: int = 0
    fillins_dense_kept: int = 0


def _perm_to_piv(perm: np.ndarray) -> np.ndarray:
    """Row permutation (row l of P S = row perm[l] of S) -> LAPACK getrf pivots
    (row l was interchanged with row piv[l], applied in order), as scipy's
    lu_factor returns them."""
    m = len(perm)
    cur = np.arange(m)
    where = np.arange(m)
    piv = np.empty(m, dtype=np.int32)
    for l in range(m):
        p = where[perm[l]]
        piv[l] = p
        a, b = cur[l], cur[p]
        cur[l], cur[p] = b, a
        where[b], where[a] = l, p
    return piv


class Record:
    """One cluster elimination (the reference's _Record, ifmm/solver.py:63-74).
    `lu` is scipy lu_factor's (lu, piv) of the pivot block S, downloaded on
    first access; z_partners equal y_partners (the stored system is symmetric:
    the local rows referencing x_i belong to the partners it couples through M2P)."""

    __slots__ = ("_fact", "_idx", "level", "index", "n", "r", "w", "x_partners", "y_partners", "_lu")

    def __init__(self, fact, idx, info, xp, yp):
        self._fact, self._idx = fact, idx
        self.level, self.index, self.n, self.r, self.w = map(int, info[:5])
        self.x_partners = [int(v) for v in xp]
        self.y_partners = [int(v) for v in yp]
        self._lu = None

    @property
    def z_partners(self) -> list:
        return list(self.y_partners)

    @property
    def lu(self) -> tuple:
        if self._lu is None:
            m = self.n + self.r
            a = np.empty((m, m))  # column-major m x m = a.T
            perm = np.empty(m, dtype=np.int32)
            _lib.check(_lib.lib.ifmm_factor_record_lu(self._fact.handle, self._idx, _lib.ptr(a), _lib.ptr(perm)))
            self._lu = (np.ascontiguousarray(a.T), _perm_to_piv(perm))
        return self._lu

    def __repr__(self):
        return (f"Record(level={self.level}, index={self.index}, n={self.n}, r={self.r}, w={self.w}, "
                f"x_partners={self.x_partners}, y_partners={self.y_partners})")


@dataclass
class IfmmFactorization:
    store: OperatorStore
    tree: ClusterTree
    tol: float
    handle: object = None
    level_stats: dict = field(default_factory=dict)
    r_m: int = 0
    top_dim: int = 0
    n_records: int = 0
    factor_ms: float = 0.0
    last_refinement: list = field(default_factory=list)
    # extension: largest pivot condition estimate per level, and (with
    # on_singular="record") every pivot over the limit as (level, index, cond)
    max_cond: dict = field(default_factory=dict)
    singular_pivots: list = field(default_factory=list)
    # extension (rank_tol): sum of the pivots' basis ranks before / after consolidation
    rank_control: tuple = (0, 0)

    @property
    def n(self) -> int:
        return self.tree.n_points

    @property
    def records(self) -> list:
        """Eliminations in order (ifmm/solver.py:63-74 _Record); a sharded
        factorization lists this rank's own."""
        out = []
        info = np.zeros(7, dtype=np.int32)
        for idx in range(self.n_records):
            _lib.check(_lib.lib.ifmm_factor_record(self.handle, idx, _lib.ptr(info), None, None))
            xp = np.zeros(max(1, int(info[5])), dtype=np.int32)
            yp = np.zeros(max(1, int(info[6])), dtype=np.int32)
            _lib.check(_lib.lib.ifmm_factor_record(self.handle, idx, _lib.ptr(info), _lib.ptr(xp), _lib.ptr(yp)))
            out.append(Record(self, idx, info.copy(), xp[:info[5]], yp[:info[6]]))
        return out

    @property
    def top_lu(self) -> tuple:
        """scipy lu_factor-style (lu, piv) of the level-2 top system (ifmm/solver.py:528-546)."""
        m = self.top_dim
        a = np.empty((m, m))
        perm = np.empty(max(1, m), dtype=np.int32)
        _lib.check(_lib.lib.ifmm_factor_top(self.handle, _lib.ptr(a), _lib.ptr(perm), None))
        return np.ascontiguousarray(a.T), _perm_to_piv(perm[:m])

    @property
    def top_offsets(self) -> np.ndarray:
        """Offsets of the level-2 clusters in the top system (IfmmFactorization.top_offsets)."""
        off = np.zeros((1 << (2 * self.tree.dim)) + 1, dtype=np.int64)
        _lib.check(_lib.lib.ifmm_factor_top(self.handle, None, None, _lib.ptr(off)))
        return off

    @property
    def work(self) -> dict:
        """Executed / reference-equivalent FP64 flops and solve bytes per rhs."""
        w = np.empty(6)
        _lib.check(_lib.lib.ifmm_factor_work(self.handle, _lib.ptr(w)))
        return {"flops_exec": w[0], "flops_schur": w[1], "flops_ref": w[2], "solve_bytes": w[3], "flops_lu": w[4],
                "flops_x": w[5]}

    @property
    def phase_times(self) -> dict:
        """Device ms and kernel launches per factorization phase (needs timing=True)."""
        ms = np.zeros(7)
        nl = np.zeros(7, dtype=np.int64)
        _lib.check(_lib.lib.ifmm_factor_timing(self.handle, _lib.ptr(ms), _lib.ptr(nl)))
        return {p: (float(ms[i]), int(nl[i])) for i, p in enumerate(PHASES)}

    @property
    def phase_times_by_level(self) -> dict:
        """{level: {phase: ms}} (level 1 = top-level inverse); needs timing=True."""
        out = {}
        for k in range(1, self.tree.depth + 1):
            ms = np.zeros(9)
            _lib.check(_lib.lib.ifmm_factor_timing_level(self.handle, k, _lib.ptr(ms)))
            if ms.any():
                out[k] = {p: round(float(ms[i]), 3) for i, p in enumerate(PHASES + ("host_busy", "host_wait"))}
        return out

    @property
    def shard(self) -> dict:
        """Sharded factorizations: this rank, the rank count and traffic
        (halo / metadata bytes sent, exchanges, device ms in communication
        with timing=True).  One GPU: rank 0 of 1, no traffic."""
        rn = np.zeros(2, dtype=np.int32)
        o = np.zeros(4)
        _lib.check(_lib.lib.ifmm_factor_shard_info(self.handle, _lib.ptr(rn), _lib.ptr(o)))
        return {"rank": int(rn[0]), "nranks": int(rn[1]), "halo_bytes": o[0], "meta_bytes": o[1],
                "exchanges": int(o[2]), "comm_ms": o[3]}

    def __del__(self):
        h, self.handle = getattr(self, "handle", None), None
        lib = getattr(_lib, "lib", None)
        if h and lib is not None:  # at interpreter shutdown the module may already be torn down
            lib.ifmm_factor_free(h)


PHASES = ("gather", "lu", "x_solve", "schur", "compress", "transition", "top")


def factorize(store: OperatorStore, tree: ClusterTree, tol: float | None = None, diagnostics: bool = False,
              release_m2l: bool = True, timing: bool = False,
              pivot_condition_limit: float = PIVOT_CONDITION_LIMIT, comm=None,
              on_singular: str = "raise", rank_tol: float | None = None) -> IfmmFactorization:
    """Eliminate the extended system on the GPU (ifmm/solver.py:106-153).

    Unlike the reference the store's initial operators stay intact (the
    elimination works on its own device copy), so `fmm_matvec(store, ...)`
    remains valid afterwards.  `release_m2l` is accepted for API parity:
    finished levels are always released.

    comm (extension): a `distributed.Communicator`; the call is then
    collective over its ranks, each eliminating its own level-2 subtrees
    (every rank passes the same store contents).

    on_singular (extension): "raise" (the reference's behaviour,
    ifmm/solver.py:214-218) raises SingularPivotError at the first pivot whose
    condition estimate exceeds `pivot_condition_limit`; "record" lists such
    pivots in `fact.singular_pivots` and carries on (sharded runs: each rank
    lists its own pivots).

    rank_tol (extension, SURVEY 8f item 3 -- rank-growth control, the
    reference's unused `_maybe_consolidate`, ifmm/solver.py:437-492): right
    before a cluster is eliminated its coupling row (its M2L blocks and its
    rows of the parent's basis) is re-truncated jointly at `rank_tol` relative
    to the row's largest singular value and the basis rotated onto the kept
    directions.  Ranks stop creeping toward the particle dimension, pivots and
    parents shrink.  None (default) keeps the reference's arithmetic;
    `fact.rank_control` = (rank sum before, after; a sharded run counts this
    rank's pivots)."""
    if on_singular not in ("raise", "record"):
        raise ValueError(f"on_singular must be 'raise' or 'record', got {on_singular!r}")
    if tol is None:
        tol = store.tol
    h = ctypes.c_void_p()
    flags = (1 if timing else 0) | (2 if on_singular == "record" else 0)
    sharded = comm is not None and comm.size > 1
    if rank_tol is not None and not 0.0 < rank_tol < 1.0:
        raise ValueError(f"rank_tol must lie in (0, 1), got {rank_tol!r}")
    if rank_tol is not None and sharded:
        _lib.check(_lib.lib.ifmm_factorize_sharded_rank_control(store.handle, comm.handle, float(tol), flags,
                                                                float(pivot_condition_limit), float(rank_tol),
                                                                ctypes.byref(h)))
    elif rank_tol is not None:
        _lib.check(_lib.lib.ifmm_factorize_rank_control(store.handle, float(tol), flags,
                                                        float(pivot_condition_limit), float(rank_tol),
                                                        ctypes.byref(h)))
    elif sharded:
        _lib.check(_lib.lib.ifmm_factorize_sharded(store.handle, comm.handle, float(tol), flags,
                                                   float(pivot_condition_limit), ctypes.byref(h)))
    else:
        _lib.check(_lib.lib.ifmm_factorize(store.handle, float(tol), flags, float(pivot_condition_limit),
                                           ctypes.byref(h)))
    fact = _wrap_factor(store, tree, float(tol), h)
    fact._comm = comm  # collective solves call back through the communicator
    if diagnostics:
        for k in range(tree.depth, 1, -1):
            s = fact.level_stats[k]
            logger.info("level=%d,k_clusters=%d,max_rank=%d,fillins_compressed=%d,fillins_dense_kept=%d",
                        k, s.clusters, s.max_rank, s.fillins_compressed, s.fillins_dense_kept)
    return fact


def _wrap_factor(store: OperatorStore, tree: ClusterTree, tol: float, h) -> IfmmFactorization:
    fact = IfmmFactorization(store=store, tree=tree, tol=tol, handle=h)
    rm, top = ctypes.c_int(), ctypes.c_int()
    nrec, ms = ctypes.c_int64(), ctypes.c_double()
    _lib.check(_lib.lib.ifmm_factor_info(h, ctypes.byref(rm), ctypes.byref(top), ctypes.byref(nrec),
                                         ctypes.byref(ms)))
    fact.r_m, fact.top_dim, fact.n_records, fact.factor_ms = rm.value, top.value, nrec.value, ms.value
    rc = np.zeros(2, dtype=np.int64)
    _lib.check(_lib.lib.ifmm_factor_rank_control(h, _lib.ptr(rc)))
    fact.rank_control = (int(rc[0]), int(rc[1]))
    for k in range(tree.depth, 1, -1):
        st = np.zeros(4, dtype=np.int32)
        _lib.check(_lib.lib.ifmm_factor_level_stats(h, k, _lib.ptr(st)))
        fact.level_stats[k] = LevelStats(*map(int, st))
        c = ctypes.c_double()
        _lib.check(_lib.lib.ifmm_factor_level_cond(h, k, ctypes.byref(c)))
        fact.max_cond[k] = c.value
    cnt = ctypes.c_int64()
    _lib.check(_lib.lib.ifmm_factor_singular(h, 0, None, None, None, ctypes.byref(cnt)))
    if cnt.value:
        lv = np.zeros(cnt.value, dtype=np.int32)
        ix = np.zeros(cnt.value, dtype=np.int32)
        cd = np.zeros(cnt.value)
        _lib.check(_lib.lib.ifmm_factor_singular(h, cnt.value, _lib.ptr(lv), _lib.ptr(ix), _lib.ptr(cd),
                                                 ctypes.byref(cnt)))
        fact.singular_pivots = [(int(a), int(b), float(c)) for a, b, c in zip(lv, ix, cd)]
    return fact


def solve(fact: IfmmFactorization, rhs, refine: int = 0, target: float = 0.0):
    """Solve the factored system (ifmm/solver.py:549-626).  `rhs` is (N,) (as
    the reference) or (N, nrhs); numpy or torch (CUDA tensors stay on device).
    Returns the solution in original point order.

    refine > 0 (extension): up to `refine` steps of iterative refinement with
    the store's compressed FMM operator, stopping once the relative residual
    ||b - A~ x|| / ||b|| <= target; the residual history is left in
    `fact.last_refinement`."""
    n = fact.tree.n_points
    if isinstance(rhs, np.ndarray) or not type(rhs).__module__.startswith("torch"):
        a = np.asarray(rhs, dtype=float)
        if a.ndim not in (1, 2) or a.shape[0] != n:
            raise ValueError(f"rhs must have shape ({n},)")
    p_in, kind, nr, keep, is_torch, one_d = _lib.as_input(rhs, n)
    out, p_out = _lib.alloc_output(keep, kind, n, nr, one_d)
    if refine > 0:
        hist = np.zeros(int(refine) + 1)
        done = ctypes.c_int()
        _lib.check(_lib.lib.ifmm_solve_refined(fact.handle, fact.store.handle, p_in, p_out, nr, kind, int(refine),
                                               float(target), _lib.ptr(hist), ctypes.byref(done)))
        fact.last_refinement = hist[:done.value + 1].tolist()
    else:
        _lib.check(_lib.lib.ifmm_solve(fact.handle, p_in, p_out, nr, kind))
    if is_torch and kind == _lib.PTR_HOST:
        import torch
        out = torch.from_numpy(out)
    return out[:, 0] if one_d else out
