"""Per-rank host time of the sharded schedule (virtual ranks on one GPU): host_busy /
host_wait summed over levels for 1 GPU and V virtual ranks.
    python tools/shard_host.py CONFIG V [V ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_1407_1572_b200 as ifmm  # noqa: E402
from paper_1407_1572_b200 import distributed as D  # noqa: E402

name = sys.argv[1]
N, kern, depth, p, tol, _ = bench.CONFIGS[name]
pts = 2.0 * np.random.default_rng(0).random((N, 2)) - 1.0
tree = ifmm.build_tree(ifmm.PointSet(2, pts), depth)
store = ifmm.init_operators(tree, ifmm.baseline_kernel(kern, N), p=p, tol=tol)


def host(f):
    lv = f.phase_times_by_level
    return sum(v["host_busy"] for v in lv.values()), sum(v["host_wait"] for v in lv.values())


f1 = ifmm.factorize(store, tree, pivot_condition_limit=np.inf, timing=True)
print(f"{name} 1 GPU: host busy {host(f1)[0]:.0f} ms, wait {host(f1)[1]:.0f} ms, factor {f1.factor_ms:.0f} ms", flush=True)
del f1
for V in [int(v) for v in sys.argv[2:]]:
    fs = D.factorize_emulated(store, tree, V, timing=True, pivot_condition_limit=np.inf)
    hb = [host(f) for f in fs]
    print(f"{name} {V} virtual ranks: host busy per rank {[round(a) for a, _ in hb]} ms, wait "
          f"{[round(b) for _, b in hb]} ms", flush=True)
    del fs
