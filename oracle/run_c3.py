"""Run the CPU oracle (the reference algorithm, bit-exact restatement) at BASELINE C3 itself.

TEST INFRASTRUCTURE ONLY (see ifmm_oracle.py header).  This is the reference's timing protocol
(`ifmm/cli.py:86-110`: t_a = init_operators, t_f = factorize, t_s = median of 3 solves, residual
against the FMM operator of a fresh store) on N = 1,048,576, 1/|x-y| with diagonal sqrt(N),
depth 7, p = 4, eps = 1e-6, one N(0,1) rhs, seed 0 -- the bench.py C3 workload.

It needs ~70 GB of RAM and about an hour on one core, so it runs on the GPU box's host
(196 GB, 16 cores), one process per elimination order:

    OMP_NUM_THREADS=1 OPENBLAS_NUM_THREADS=1 python oracle/run_c3.py morton  gpurun_out/c3
    OMP_NUM_THREADS=1 OPENBLAS_NUM_THREADS=1 python oracle/run_c3.py colour9 gpurun_out/c3

The reference raises SingularPivotError when a pivot's 1-norm condition estimate exceeds 1e12
(`ifmm/solver.py:50,214-218`).  The run records every such pivot instead of stopping
(`on_singular="record"`), so one run answers both "does the reference itself trip at C3" (the
first recorded pivot is where it would raise) and "what does it compute if it does not".
`oracle/make_c3_golden.py` turns the two outputs into tests/golden/c3_1m.npz.
"""
import json
import os
import resource
import sys
import threading
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle import ifmm_oracle as O  # noqa: E402

RSS_GUARD_GB = float(os.environ.get("C3_RSS_GUARD_GB", "92"))


def rss_gb():
    with open("/proc/self/status") as f:
        for line in f:
            if line.startswith("VmRSS:"):
                return int(line.split()[1]) / 2**20
    return 0.0


def peak_gb():
    return resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 2**20


def main():
    order = sys.argv[1]
    out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/c3"
    n_arg = int(sys.argv[3]) if len(sys.argv) > 3 else 1048576
    depth = {1048576: 7, 262144: 6, 65536: 5, 16384: 4}[n_arg]
    os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
    log = open(f"{out}_{order}.log", "w")

    def say(msg):
        line = f"[{time.strftime('%H:%M:%S')}] {msg} (rss {rss_gb():.1f} GB)"
        print(line, flush=True)
        log.write(line + "\n")
        log.flush()

    def guard():
        while True:
            if rss_gb() > RSS_GUARD_GB:
                say(f"RSS guard {RSS_GUARD_GB} GB tripped: not completed")
                os._exit(3)
            time.sleep(2.0)
    threading.Thread(target=guard, daemon=True).start()

    N, kern, p, tol = n_arg, "inv_r", 4, 1e-6
    say(f"C3 oracle run: N={N} kernel={kern} depth={depth} p={p} tol={tol} order={order} "
        f"affinity={len(os.sched_getaffinity(0))} cores, host cpus={os.cpu_count()}, "
        f"BLAS threads={os.environ.get('OPENBLAS_NUM_THREADS')}")
    pts = O.baseline_points(N, seed=0)
    spec = O.baseline_kernel(kern, N)
    b = O.baseline_rhs(N, "normal")
    t0 = time.perf_counter()
    tree = O.build_tree(pts, depth)
    t_tree = time.perf_counter() - t0
    t0 = time.perf_counter()
    st = O.init_operators(tree, spec, p, tol)
    t_a = time.perf_counter() - t0
    say(f"tree {t_tree:.1f}s  init_operators t_a {t_a:.1f}s")
    lvl_t = {}
    t_start = time.perf_counter()

    def progress(k, fac):
        lvl_t[k] = time.perf_counter() - t_start
        s = fac.stats[k]
        say(f"level {k} done at {lvl_t[k]:.1f}s: compressed {s.compressed} dense_kept {s.dense_kept} "
            f"max_rank {s.max_rank} max_cond {fac.max_cond.get(k, 0):.3e} singular so far {len(fac.singular)}")

    t0 = time.perf_counter()
    fac = O.factorize(st, tol, order=order, on_singular="record", progress=progress)
    t_f = time.perf_counter() - t0
    top = int(fac.top_off[-1])
    say(f"factorize t_f {t_f:.1f}s  top {top}  r_m {fac.r_m}  singular pivots {len(fac.singular)}"
        + (f" first {fac.singular[0]}" if fac.singular else ""))
    ts = []
    x = None
    for _ in range(3):
        t0 = time.perf_counter()
        x = O.solve(fac, b)
        ts.append(time.perf_counter() - t0)
    t_s = float(np.median(ts))
    say(f"solve t_s {t_s:.2f}s (median of 3)")
    stats = np.array([[k, s.clusters, s.max_rank, s.compressed, s.dense_kept]
                      for k, s in sorted(fac.stats.items())], dtype=np.int64)
    rank_sum = {k: int(sum(st.r(k, i) for i in range(tree.n_clusters(k)))) for k in range(2, depth + 1)}
    singular = np.array(fac.singular, dtype=float).reshape(-1, 3)
    max_cond = np.array([[k, c] for k, c in sorted(fac.max_cond.items())])
    r_m = fac.r_m
    peak_fact = peak_gb()
    del fac, st
    st2 = O.init_operators(tree, spec, p, tol)
    resid = float(np.linalg.norm(O.fmm_matvec(st2, x) - b) / np.linalg.norm(b))
    say(f"residual vs FMM operator {resid:.3e}")
    np.savez_compressed(f"{out}_{order}.npz", x=x, perm=tree.perm.astype(np.int32),
                        leaf_off=tree.leaf_off.astype(np.int64), stats=stats, top=top, r_m=r_m,
                        resid=resid, singular=singular, max_cond=max_cond,
                        rank_sum=np.array(sorted(rank_sum.items()), dtype=np.int64))
    summary = dict(order=order, N=N, depth=depth, p=p, tol=tol, kernel=kern, t_tree=t_tree, t_a=t_a,
                   t_f=t_f, t_s=t_s, t_s_all=ts, level_done_s=lvl_t, top=top, r_m=r_m, resid=resid,
                   singular_count=len(singular), first_singular=singular[0].tolist() if len(singular) else None,
                   max_cond={int(k): float(c) for k, c in max_cond}, peak_rss_gb_factor=peak_fact,
                   peak_rss_gb=peak_gb(), cores_used=1, host_cpus=os.cpu_count(),
                   blas_threads=os.environ.get("OPENBLAS_NUM_THREADS"))
    with open(f"{out}_{order}.json", "w") as f:
        json.dump(summary, f, indent=1)
    say("done " + json.dumps(summary))


if __name__ == "__main__":
    main()
