"""CPU checks of the subtree-sharded path -- no GPU needed.

* the partition (owner / held tables, csrc/comm.cu make_partition) against its
  definition: level-2 subtrees dealt in contiguous Morton ranges, children
  inherit the owner, a rank stores its own clusters and their neighbours,
  every rank stores level 2;
* a world-size-2 gloo job: the NCCL unique id broadcast the Python side uses,
  and the halo routing rule (comm.cuh halo_route, the one the factorization
  runs) evaluated independently on each rank -- what rank a plans to send to b
  must equal what b plans to receive from a, for every level and colour batch.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _grid(k, dim=2):
    i = np.arange(1 << (dim * k))
    g = np.zeros((i.size, dim), dtype=np.int64)
    for b in range(k):
        for ax in range(dim):
            g[:, ax] |= ((i >> (b * dim + ax)) & 1) << b
    return g


@pytest.mark.parametrize("nranks", [1, 2, 3, 4, 8, 16])
def test_partition_definition(nranks):
    from paper_1407_1572_b200 import distributed as D
    depth = 5
    for k in range(2, depth + 1):
        owner, held = D.partition(depth, k, nranks)
        nc = 1 << (2 * k)
        assert owner.shape == (nc,) and held.shape == (nranks, nc)
        # contiguous Morton ranges of level-2 subtrees
        anc = np.arange(nc) >> (2 * (k - 2))
        assert np.array_equal(owner, (anc * nranks) // 16)
        assert set(owner.tolist()) == set(range(nranks))
        if k > 2:
            po, _ = D.partition(depth, k - 1, nranks)
            assert np.array_equal(owner, po[np.arange(nc) >> 2]), "children inherit the owner"
        g = _grid(k)
        cheb = np.abs(g[:, None, :] - g[None, :, :]).max(axis=2)
        for s in range(nranks):
            if k == 2:
                assert held[s].all()
                continue
            want = (cheb[:, owner == s] <= 1).any(axis=1)
            assert np.array_equal(held[s], want), (k, s)


def test_partition_rejects_too_many_ranks():
    from paper_1407_1572_b200 import distributed as D
    with pytest.raises(ValueError, match="ranks"):
        D.partition(4, 3, 17)


def _counts(depth, level, nranks, rank, colour):
    import ctypes
    from paper_1407_1572_b200 import _lib
    s = np.zeros(nranks, dtype=np.int32)
    r = np.zeros(nranks, dtype=np.int32)
    _lib.check(_lib.lib.ifmm_partition_halo_counts(2, depth, level, nranks, rank, colour, _lib.ptr(s), _lib.ptr(r)))
    return s, r


@pytest.mark.parametrize("nranks", [2, 4, 8])
def test_halo_plan_matches_between_ranks_single_process(nranks):
    depth = 5
    for level in range(2, depth + 1):
        for colour in range(9):
            plans = [_counts(depth, level, nranks, q, colour) for q in range(nranks)]
            for a in range(nranks):
                for b in range(nranks):
                    if a != b:
                        assert plans[a][0][b] == plans[b][1][a], (level, colour, a, b)
                assert plans[a][0][a] == 0 and plans[a][1][a] == 0
            if level > 2 and nranks > 1:
                assert sum(p[0].sum() for p in plans) > 0  # boundary pivots do ship something


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_1407_1572_b200 import distributed as D
        uid = D.broadcast_unique_id()
        ids = [None] * world
        dist.all_gather_object(ids, uid)
        ok_id = len(uid) == 128 and all(x == uid for x in ids)
        # each rank evaluates the routing rule for itself; gather and cross-check
        depth, mism, total = 6, 0, 0
        plans = {}
        for level in range(2, depth + 1):
            for colour in range(9):
                plans[(level, colour)] = [c.tolist() for c in _counts(depth, level, world, rank, colour)]
        allp = [None] * world
        dist.all_gather_object(allp, plans)
        for key in plans:
            for a in range(world):
                for b in range(world):
                    if a != b:
                        total += allp[a][key][0][b]
                        mism += allp[a][key][0][b] != allp[b][key][1][a]
        owner, held = D.partition(depth, depth, world)
        owned = [None] * world
        dist.all_gather_object(owned, np.flatnonzero(owner == rank).tolist())
        cover = sorted(sum(owned, [])) == list(range(owner.size))
        q.put((rank, ok_id, mism, total, cover))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e), -1, 0, False))


def test_gloo_world2_id_broadcast_and_halo_plan():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, ok_id, mism, total, cover in res:
        assert ok_id is True, ok_id
        assert mism == 0 and total > 0, (rank, mism, total)
        assert cover
