"""One rank of the host-transport test (tests/test_gpu_sharded.py::test_two_processes_host_transport):
launched by torch.distributed.run with the gloo backend, every rank drives the same GPU and factorizes
ONE system together through the host-staged communicator; rank 0 saves the solution.

    python -m torch.distributed.run --nproc-per-node 2 ... tests/host_transport_worker.py OUT.npz N DEPTH KERNEL P TOL [RANK_TOL]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1407_1572_b200 as ifmm  # noqa: E402
from paper_1407_1572_b200.distributed import Communicator  # noqa: E402

out, n, depth, kern, p, tol = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], int(sys.argv[5]), \
    float(sys.argv[6])
rank_tol = float(sys.argv[7]) if len(sys.argv) > 7 else None
dist.init_process_group("gloo")
pts = 2.0 * np.random.default_rng(0).random((n, 2)) - 1.0
b = np.random.default_rng([0, 1]).standard_normal(n)
tree = ifmm.build_tree(ifmm.PointSet(2, pts), depth)
store = ifmm.init_operators(tree, ifmm.baseline_kernel(kern, n), p=p, tol=tol)
comm = Communicator.host()
fact = ifmm.factorize(store, tree, comm=comm, pivot_condition_limit=np.inf, rank_tol=rank_tol)
x = ifmm.solve(fact, b)
sh = fact.shard
if dist.get_rank() == 0:
    np.savez(out, x=x, top=fact.top_dim, halo=sh["halo_bytes"], exchanges=sh["exchanges"], nrec=fact.n_records)
dist.barrier()
dist.destroy_process_group()
