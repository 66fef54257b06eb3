"""Device memory of one factorization (cudaMemGetInfo around factorize), per config.
    python tools/mem_probe.py C3 [C3_262k C5_4m:1e-7 ...]     (NAME:rank_tol = with rank-growth control)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1407_1572_b200 as ifmm  # noqa: E402

import time  # noqa: E402

for arg in sys.argv[1:]:
    name, _, rt = arg.partition(":")
    rt = float(rt) if rt else None
    N, kern, depth, p, tol, nrhs = bench.CONFIGS[name]
    pts = 2.0 * np.random.default_rng(0).random((N, 2)) - 1.0
    free0, total = torch.cuda.mem_get_info()
    tree = ifmm.build_tree(ifmm.PointSet(2, pts), depth)
    store = ifmm.init_operators(tree, ifmm.baseline_kernel(kern, N), p=p, tol=tol)
    free1, _ = torch.cuda.mem_get_info()
    t0 = time.perf_counter()
    f = ifmm.factorize(store, tree, on_singular="record", pivot_condition_limit=np.inf, rank_tol=rt)
    t1 = time.perf_counter()
    free2, _ = torch.cuda.mem_get_info()
    print(f"{arg}: factorize {t1 - t0:.2f} s, top {f.top_dim}, rank control {f.rank_control}")
    print(f"{name}: N={N} store {(free0 - free1) / 1e9:.1f} GB, after factorize {(free0 - free2) / 1e9:.1f} GB in use "
          f"(device total {total / 1e9:.0f} GB); records {f.n_records}, solve bytes {f.work['solve_bytes'] / 1e9:.1f} GB",
          flush=True)
    del f, store, tree
