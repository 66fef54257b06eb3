"""Subtree-sharded factorize / solve over several GPUs.

The reference (`ifmm/solver.py`) is one process on one CPU; it has no
distributed path.  Here one process drives one GPU and the quadtree is split by
level-2 subtrees (2 ranks: halves, 4: quadrants, 8: pairs of level-2 cells, in
Morton order); every rank replays the host schedule of `factorize`
(ifmm/solver.py:106-153, colour-batched), eliminates its own subtrees' clusters
and, after each colour batch, ships the blocks it wrote to the ranks that store
them (its neighbours within one cell) with NCCL send/recv over NVLink.  The
level-2 system is held by every rank and inverted on each.  `solve` on a
sharded factorization is collective and returns the full solution on every rank.

    comm = Communicator.from_torch()          # after torch.distributed.init_process_group
    fact = factorize(store, tree, comm=comm)  # paper_1407_1572_b200.factorize
    x = solve(fact, b)                        # same b on every rank

`factorize_emulated` runs the same schedule with V virtual ranks as threads on
one GPU (device-to-device copies instead of NCCL) -- the single-GPU check of
the sharded schedule used by the tests.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib

__all__ = ["Communicator", "partition", "factorize_emulated", "solve_emulated", "max_ranks"]


def max_ranks(dim: int = 2) -> int:
    """Ranks the subtree partition supports: one per level-2 cluster at most."""
    return 1 << (2 * dim)


def partition(depth: int, level: int, nranks: int, dim: int = 2):
    """(owner[nc], held[nranks, nc]) of the clusters of `level` (host-only)."""
    nc = 1 << (dim * level)
    owner = np.zeros(nc, dtype=np.int32)
    held = np.zeros((nranks, nc), dtype=np.uint8)
    _lib.check(_lib.lib.ifmm_partition(dim, depth, level, nranks, _lib.ptr(owner), _lib.ptr(held)))
    return owner, held.astype(bool)


def broadcast_unique_id(group=None) -> bytes:
    """Rank 0 of `group` creates an NCCL unique id; torch.distributed (any
    backend) broadcasts it to the other ranks."""
    import torch.distributed as dist
    obj = [Communicator.unique_id() if dist.get_rank(group) == 0 else None]
    src = 0 if group is None else dist.get_global_rank(group, 0)
    dist.broadcast_object_list(obj, src=src, group=group)
    return obj[0]


_P = ctypes.POINTER
_HOST_AG = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64)
_HOST_EX = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int, _P(ctypes.c_int32), _P(ctypes.c_void_p),
                            _P(ctypes.c_int64), ctypes.c_int, _P(ctypes.c_int32), _P(ctypes.c_void_p),
                            _P(ctypes.c_int64))


class Communicator:
    """NCCL communicator of the library (one rank per process / GPU)."""

    def __init__(self, handle, rank: int, size: int):
        self.handle = handle
        self.rank = rank
        self.size = size

    @staticmethod
    def unique_id() -> bytes:
        buf = (ctypes.c_uint8 * 128)()
        _lib.check(_lib.lib.ifmm_comm_nccl_unique_id(ctypes.cast(buf, ctypes.c_void_p)))
        return bytes(buf)

    @classmethod
    def nccl(cls, unique_id: bytes, nranks: int, rank: int) -> "Communicator":
        """Collective: every rank passes the same 128-byte id."""
        if len(unique_id) != 128:
            raise ValueError("NCCL unique id must be 128 bytes")
        if not 0 <= rank < nranks:
            raise ValueError(f"rank {rank} out of range for {nranks} ranks")
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(unique_id)
        h = ctypes.c_void_p()
        _lib.check(_lib.lib.ifmm_comm_nccl_init(ctypes.cast(buf, ctypes.c_void_p), int(nranks), int(rank),
                                                ctypes.byref(h)))
        return cls(h, rank, nranks)

    @classmethod
    def from_torch(cls, group=None) -> "Communicator":
        """Collective over a torch.distributed process group: rank 0 creates the
        NCCL id, torch broadcasts it, every rank joins (its current CUDA device)."""
        import torch.distributed as dist
        rank, size = dist.get_rank(group), dist.get_world_size(group)
        return cls.nccl(broadcast_unique_id(group), size, rank)

    @classmethod
    def host(cls, group=None) -> "Communicator":
        """Collective over a torch.distributed group of ANY backend (gloo on
        CPU tensors): the library's collectives are staged through pinned host
        memory and handed to torch.distributed (all_gather, isend / irecv).
        Slow; it runs the real multi-process schedule on processes that share
        one GPU, where NCCL refuses duplicate devices."""
        import torch
        import torch.distributed as dist
        rank, size = dist.get_rank(group), dist.get_world_size(group)
        glob = (lambda r: r) if group is None else (lambda r: dist.get_global_rank(group, r))

        def view(addr, n):
            return np.ctypeslib.as_array((ctypes.c_uint8 * n).from_address(addr)) if n else np.zeros(0, np.uint8)

        def allgather(ctx, send, recv, nbytes):
            try:
                t = torch.from_numpy(view(send, nbytes).copy())
                outs = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(size)]
                dist.all_gather(outs, t, group=group)
                dst = view(recv, nbytes * size)
                for q, o in enumerate(outs):
                    dst[q * nbytes:(q + 1) * nbytes] = o.numpy()
                return 0
            except Exception:  # pragma: no cover - reported as a library error
                import traceback
                traceback.print_exc()
                return 1

        def exchange(ctx, ns, sp, sb, sn, nr, rp, rb, rn):
            try:
                reqs, keep, tags = [], [], {}
                # zero-byte messages are not sent (as with NCCL); the k-th nonzero
                # message between a pair carries tag k on both sides
                for i in range(ns):
                    if sn[i] == 0:
                        continue
                    tag = tags.get(("s", sp[i]), 0)
                    tags[("s", sp[i])] = tag + 1
                    t = torch.from_numpy(view(sb[i], sn[i]).copy())
                    keep.append(t)
                    reqs.append(dist.isend(t, dst=glob(sp[i]), group=group, tag=tag))
                outs = []
                for i in range(nr):
                    if rn[i] == 0:
                        continue
                    tag = tags.get(("r", rp[i]), 0)
                    tags[("r", rp[i])] = tag + 1
                    t = torch.empty(rn[i], dtype=torch.uint8)
                    outs.append((i, t))
                    reqs.append(dist.irecv(t, src=glob(rp[i]), group=group, tag=tag))
                for r in reqs:
                    r.wait()
                for i, t in outs:
                    view(rb[i], rn[i])[:] = t.numpy()
                return 0
            except Exception:  # pragma: no cover
                import traceback
                traceback.print_exc()
                return 1

        cb_ag, cb_ex = _HOST_AG(allgather), _HOST_EX(exchange)
        h = ctypes.c_void_p()
        _lib.check(_lib.lib.ifmm_comm_host_init(int(size), int(rank), ctypes.cast(cb_ag, ctypes.c_void_p),
                                                ctypes.cast(cb_ex, ctypes.c_void_p), None, ctypes.byref(h)))
        c = cls(h, rank, size)
        c._callbacks = (cb_ag, cb_ex)  # the library holds raw pointers to them
        return c

    def selftest(self, n: int = 4096) -> bool:
        """Collective: all-gather + ring send/recv of n doubles through the library's transport."""
        ok = ctypes.c_int32()
        _lib.check(_lib.lib.ifmm_comm_selftest(self.handle, int(n), ctypes.byref(ok)))
        return bool(ok.value)

    def __del__(self):
        h, self.handle = getattr(self, "handle", None), None
        lib = getattr(_lib, "lib", None)
        if h and lib is not None:
            lib.ifmm_comm_free(h)  # factorizations keep their own reference


def factorize_emulated(store, tree, nranks: int, tol: float | None = None, timing: bool = False,
                       pivot_condition_limit: float = 1e12, rank_tol: float | None = None) -> list:
    """The sharded schedule with `nranks` virtual ranks on the current GPU;
    returns one IfmmFactorization per rank."""
    from .solver import _wrap_factor
    if tol is None:
        tol = store.tol
    hs = (ctypes.c_void_p * nranks)()
    if rank_tol is not None:
        _lib.check(_lib.lib.ifmm_factorize_emulated_rank_control(
            store.handle, int(nranks), float(tol), 1 if timing else 0, float(pivot_condition_limit), float(rank_tol),
            ctypes.cast(hs, ctypes.c_void_p)))
    else:
        _lib.check(_lib.lib.ifmm_factorize_emulated(store.handle, int(nranks), float(tol), 1 if timing else 0,
                                                    float(pivot_condition_limit), ctypes.cast(hs, ctypes.c_void_p)))
    return [_wrap_factor(store, tree, float(tol), ctypes.c_void_p(h)) for h in hs]


def solve_emulated(facts: list, rhs) -> np.ndarray:
    """Solve on every virtual rank; returns (nranks, N[, nrhs]) solutions."""
    n = facts[0].tree.n_points
    a = np.ascontiguousarray(np.asarray(rhs, dtype=float))
    if a.ndim not in (1, 2) or a.shape[0] != n:
        raise ValueError(f"rhs must have shape ({n},) or ({n}, k)")
    nr = 1 if a.ndim == 1 else a.shape[1]
    out = np.empty((len(facts), n, nr))
    hs = (ctypes.c_void_p * len(facts))(*[f.handle.value for f in facts])
    _lib.check(_lib.lib.ifmm_solve_emulated(ctypes.cast(hs, ctypes.c_void_p), len(facts), _lib.ptr(a),
                                            _lib.ptr(out), nr, _lib.PTR_HOST))
    return out[:, :, 0] if a.ndim == 1 else out
