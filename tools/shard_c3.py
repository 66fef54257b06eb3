"""Sharded factorization of a bench config with V virtual ranks on one GPU
(LocalComm threads): solution vs the single-GPU one (must be bit-identical) and
the halo / metadata traffic per rank -- the volume NCCL would move over NVLink.

    python tools/shard_c3.py [CONFIG] [V ...]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_1407_1572_b200 as ifmm  # noqa: E402
from paper_1407_1572_b200 import distributed as D  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
ranks = [int(v) for v in sys.argv[2:]] or [8]
N, kern, depth, p, tol, _ = bench.CONFIGS[name]
pts = 2.0 * np.random.default_rng(0).random((N, 2)) - 1.0
b = np.random.default_rng([0, 1]).standard_normal(N)
tree = ifmm.build_tree(ifmm.PointSet(2, pts), depth)
store = ifmm.init_operators(tree, ifmm.baseline_kernel(kern, N), p=p, tol=tol)
ref = f"/tmp/shard_ref_{name}.npz"
if not os.path.exists(ref):  # the single-GPU solution, computed in its own process (memory)
    if os.environ.get("SHARD_SINGLE") != "1":
        import subprocess
        subprocess.run([sys.executable, __file__, name], env=dict(os.environ, SHARD_SINGLE="1"), check=True)
    else:
        f1 = ifmm.factorize(store, tree, pivot_condition_limit=1e15)
        np.savez(ref, x=ifmm.solve(f1, b), nrec=f1.n_records)
        sys.exit(0)
g = np.load(ref)
x1, nrec1 = g["x"], int(g["nrec"])
for V in ranks:
    t0 = time.perf_counter()
    fs = D.factorize_emulated(store, tree, V, pivot_condition_limit=1e15)
    t1 = time.perf_counter()
    xs = D.solve_emulated(fs, b)
    same = all(np.array_equal(xs[r], x1) for r in range(V))
    halo = [f.shard["halo_bytes"] for f in fs]
    meta = [f.shard["meta_bytes"] for f in fs]
    print(f"{name} V={V}: bit-identical to 1 GPU: {same}; records {sum(f.n_records for f in fs)} (1 GPU {nrec1}); "
          f"halo sent per rank max {max(halo) / 1e9:.2f} GB mean {np.mean(halo) / 1e9:.2f} GB; "
          f"metadata per rank {max(meta) / 1e6:.1f} MB; exchanges {fs[0].shard['exchanges']}; "
          f"emulated wall {t1 - t0:.1f} s", flush=True)
    del fs
