#!/usr/bin/env python
"""IFMM factorize + solve benchmark on B200 (BASELINE.json metric:
"IFMM factor+solve seconds at N=1M 2D; FP64 TFLOP/s vs peak; rel. residual").

A step = one factorization of the assembled extended system + one solve of
a seeded N(0,1) right-hand side (the workload BASELINE.json's metric is quoted
on: config C3, N = 1,048,576 uniform points, K = 1/|x-y| with diagonal sqrt(N),
quadtree depth 7, Chebyshev p = 4, eps = 1e-6).  Synthetic seeded data.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl reference]

Own arm: tree + operators are built once (assembly, reported with its HBM
roofline), then W warm-up and K timed steps with inputs resident in HBM (value,
ms_per_step); e2e repeats the step through the public API with host numpy
buffers (H2D rhs, D2H x inside the timed region).  The pivot-condition test is
the reference's (1e12, ifmm/solver.py:50); C3 lies past it for the reference
itself (tests/golden/c3_1m.npz: 1 pivot over the limit in Morton order, 3 in
colour order), so steps record such pivots (factorize(on_singular="record"))
and the line reports them beside the reference's counts.
--gpus N > 1 spawns N ranks (torch.distributed.run) unless already launched
under torchrun; the ranks factorize ONE system together: the subtree-sharded
path (paper_1407_1572_b200.distributed) with NCCL halo exchanges
after every colour batch -- strong scaling, timing is the max over ranks.
--impl reference times the reference algorithm (the CPU oracle restatement,
Morton order, bit-exact with /root/reference) on a bounded sample on rank 0.
"""
import argparse
import json
import math
import os
import socket
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

CONFIGS = {
    # name: N, kernel, depth, p, tol, nrhs
    "C1": (4096, "inv_r", 3, 4, 1e-8, 1),
    "C2": (65536, "log_r", 5, 5, 1e-6, 1),
    "C3": (1048576, "inv_r", 7, 4, 1e-6, 1),
    "C3_65k": (65536, "inv_r", 5, 4, 1e-6, 1),
    "C3_262k": (262144, "inv_r", 6, 4, 1e-6, 1),
    # BASELINE C5: 32 simultaneous rhs; sized for 8 GPUs (records alone ~0.85 TB)
    "C5": (16777216, "log_r", 9, 4, 1e-6, 32),
    # C5's parameters (log r, p 4, eps 1e-6, 32 rhs) at the largest size one B200 holds
    "C5_1m": (1048576, "log_r", 7, 4, 1e-6, 32),
    # C5's parameters at a quarter of C5 (two of its eight shards) on one B200: fits only with
    # rank-growth control (RANK_TOL below), which this config's factorizations therefore use
    "C5_4m": (4194304, "log_r", 8, 4, 1e-6, 32),
    # BASELINE C4's input and parameters (16-component Gaussian mixture, std 0.05, clipped; p 6, eps 1e-10)
    # on a UNIFORM depth-8 tree whose empty cells are accepted (build_tree(allow_empty_leaves=True)) -- not
    # the adaptive tree C4 names; runs with rank-growth control (without it the bases of
    # the sparse clusters run out of memory)
    "C4": (1048576, "inv_r", 8, 6, 1e-10, 1),
    "C4_65k": (65536, "inv_r", 6, 6, 1e-10, 1),
}
MIXTURE = {"C4", "C4_65k"}  # configs whose points are the C4 mixture (the others: uniform)
# configs whose timed factorizations run with rank-growth control (extension, csrc/consolidate.cu)
# (C5 itself: 2.1M points per GPU at 8 GPUs only fit with it, like C5_4m on one)
RANK_TOL = {"C5_4m": 1e-7, "C5": 1e-7, "C4": 1e-9, "C4_65k": 1e-9}
METRIC = "IFMM factor+solve seconds at N=1M 2D"
PIVOT_LIMIT = 1e12  # ifmm/solver.py:50
# bounded CPU sample of the reference algorithm: the config's parameters at a
# smaller N (depth 4 = 256 leaves of 64 points), about 9 s of one core
SAMPLE = {"C3": (16384, 4), "C3_65k": (16384, 4), "C3_262k": (16384, 4), "C2": (16384, 4), "C1": (4096, 3),
          "C5": (16384, 4), "C5_1m": (16384, 4), "C5_4m": (16384, 4), "C4": (16384, 4), "C4_65k": (16384, 4)}
C3_FULL_RUN = os.path.join(ROOT, "profiles", "r02_c3_reference_cpu.json")


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def mixture_points(n, seed=0, comps=16, std=0.05):
    """BASELINE config 4's input: a seeded 16-component isotropic Gaussian mixture in [0,1]^2 (means uniform,
    std 0.05, clipped to the box; exact duplicates -- clipping piles points onto corners -- redrawn), mapped
    to the reference box [-1,1]^2."""
    rng = np.random.default_rng(seed)
    means = rng.random((comps, 2))
    pts = np.empty((0, 2))
    while len(pts) < n:
        c = rng.integers(0, comps, n)
        x = np.clip(means[c] + std * rng.standard_normal((n, 2)), 0.0, 1.0)
        pts = np.unique(np.concatenate([pts, x]), axis=0)
    pts = pts[rng.permutation(len(pts))[:n]]
    return 2.0 * pts - 1.0


def spawn_ranks(n):
    """Re-launch this command as n ranks (one process per GPU) over 127.0.0.1."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                vals = [v.strip() for v in out.stdout.strip().split(",")]
                if len(vals) == 7:
                    self.rows.append(vals)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def measured_fp64_peak():
    """cuBLAS DGEMM 8192^3 (torch.matmul float64), best of 5: the FP64 roofline
    denominator (MEASURED_PEAKS.json carries no FP64 figure)."""
    import torch
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn_like(a)
    for _ in range(2):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    torch.cuda.empty_cache()
    return 2.0 * n ** 3 / (best * 1e-3) / 1e12


def hbm_peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]), "MEASURED_PEAKS.json"
    except Exception:
        return 6650.0, "fallback B200_PROFILING.md"


def oracle_step_seconds(n, depth, p, tol, kernel, order="morton"):
    """Reference algorithm (oracle restatement, bit-exact with the reference)
    factor + solve on one core; returns (t_factor, t_solve)."""
    from threadpoolctl import threadpool_limits
    from oracle import ifmm_oracle as O
    with threadpool_limits(1):
        pts = O.baseline_points(n, seed=0)
        spec = O.baseline_kernel(kernel, n)
        T = O.build_tree(pts, depth)
        st = O.init_operators(T, spec, p, tol)
        b = O.baseline_rhs(n, "normal")
        t0 = time.perf_counter()
        fac = O.factorize(st, tol, order=order, on_singular="record")
        t1 = time.perf_counter()
        O.solve(fac, b)
        t2 = time.perf_counter()
    return t1 - t0, t2 - t1


def c3_full_run():
    """The reference algorithm run once at C3 itself on a GPU box's host (committed log)."""
    try:
        d = json.load(open(C3_FULL_RUN))
    except Exception:
        return None
    m = d["morton"]
    return {"seconds": m["t_f"] + m["t_s"], "t_factor_s": m["t_f"], "t_solve_s": m["t_s"],
            "peak_rss_gb": m["peak_rss_gb"], "cores": m["cores_used"], "host_cpus": m["host_cpus"],
            "pivots_over_1e12": m["singular_count"], "residual": m["resid"],
            "source": os.path.relpath(C3_FULL_RUN, ROOT) + " (oracle/run_c3.py, Morton order, one core, "
                                                         "measured once; too long for a bench step)"}


def sample_desc(cfg_name, ns, ds):
    N, kern, depth, p, tol, nrhs = CONFIGS[cfg_name]
    return (f"reference algorithm (oracle/ifmm_oracle.py, Morton order, bit-exact with the reference) factor + "
            f"solve of {cfg_name}'s parameters ({kern}, p={p}, eps={tol:g}) at N={ns}, depth {ds}; one core, one "
            f"BLAS thread (the reference is a sequential elimination; multi-threaded BLAS is 4x slower on it, "
            f"SURVEY finding 8); measured, not scaled")


def run_reference(args, cfg):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    N, kern, depth, p, tol, nrhs = cfg
    ns, ds = SAMPLE[args.config]
    vals = []
    for it in range(args.warmup + args.steps):
        tf, ts = oracle_step_seconds(ns, ds, p, tol, kern)
        if it >= args.warmup:
            vals.append(tf + ts)
    v = float(np.mean(vals))
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": v * 1e3, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded uniform points, N(0,1) rhs)",
        "config": {"workload": f"{args.config} bounded sample: N={ns}, depth {ds}", "N": ns, "kernel": kern,
                   "depth": ds, "p": p, "eps": tol, "parallelism": "cpu, 1 core",
                   "note": f"each step is the bounded CPU sample; the full {args.config} system is not run per step"},
        "cpu_baseline": {"value": v, "unit": "s", "cores": 1, "kind": "port", "sample": sample_desc(args.config, ns, ds)},
        "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if args.config == "C3":
        line["c3_full_run"] = c3_full_run()
    print(json.dumps(line), flush=True)


def event_ms(fn, reps=3):
    import torch
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--rank-tol", type=float, default=None,
                    help="run the timed factorizations with rank-growth control at this tolerance (extension; "
                         "default: the reference-parity path, except for the configs in RANK_TOL)")
    ap.add_argument("--transport", default="nccl", choices=["nccl", "host"],
                    help="N > 1: NCCL (one GPU per rank), or host-staged over gloo (ranks may share a GPU; "
                         "validates the multi-process path, not a performance mode)")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    ws, rank, local = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    if ws != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}")
    if args.impl == "reference":
        run_reference(args, cfg)
        return

    import torch
    import torch.distributed as dist

    import paper_1407_1572_b200 as ifmm
    from paper_1407_1572_b200 import _lib

    if ws > 1:
        dev = local % torch.cuda.device_count()
        torch.cuda.set_device(dev)
        _lib.check(_lib.lib.ifmm_set_device(dev))
        dist.init_process_group("nccl" if args.transport == "nccl" else "gloo")
    N, kern, depth, p, tol, nrhs = cfg
    sparse = args.config in MIXTURE
    if sparse:
        pts = mixture_points(N)
    else:
        pts = 2.0 * np.random.default_rng(0).random((N, 2)) - 1.0      # [0,1]^2 mapped to the reference box
    kernel = ifmm.baseline_kernel(kern, N)
    b_host = np.random.default_rng([0, 1]).standard_normal((N, nrhs) if nrhs > 1 else N)
    b_dev = torch.from_numpy(b_host).cuda()

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tree = ifmm.build_tree(ifmm.PointSet(2, pts), depth, allow_empty_leaves=sparse)
    t1 = time.perf_counter()
    store = ifmm.init_operators(tree, kernel, p=p, tol=tol)
    t2 = time.perf_counter()
    t_tree, t_assembly = t1 - t0, t2 - t1

    comm = None
    if ws > 1:
        from paper_1407_1572_b200.distributed import Communicator
        comm = Communicator.from_torch() if args.transport == "nccl" else Communicator.host()

    rt_main = args.rank_tol if args.rank_tol is not None else RANK_TOL.get(args.config)  # None: the parity path

    def factor(timing=False):
        return ifmm.factorize(store, tree, pivot_condition_limit=PIVOT_LIMIT, on_singular="record", comm=comm,
                              timing=timing, rank_tol=rt_main)

    def step(rhs):
        fact = factor()
        return fact, ifmm.solve(fact, rhs)

    for _ in range(max(1, args.warmup)):
        fact, x = step(b_dev)
        del fact
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = _lib.lib.ifmm_launch_count()
    times = []
    with ClockSampler(local) as clk:
        for it in range(args.steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            fact, x = step(b_dev)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3)
            if it != args.steps - 1:
                del fact
    launches = (_lib.lib.ifmm_launch_count() - l0) // max(1, args.steps)
    if ws > 1:
        dist.barrier()
    t_step = float(np.mean(times))
    red_dev = "cuda" if args.transport == "nccl" else "cpu"
    if ws > 1:
        t_max = torch.tensor([t_step], device=red_dev)
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
        t_step = float(t_max.item())

    # accuracy of the last step: residual against the compressed operator
    r = ifmm.fmm_matvec(store, tree, x.double()) - b_dev
    resid = float(torch.linalg.norm(r) / torch.linalg.norm(b_dev))
    singular = list(fact.singular_pivots)
    max_cond = {int(k): v for k, v in fact.max_cond.items()}

    # extension: iterative refinement with the FMM operator to the north_star
    # accuracy (10 eps relative residual); timed separately from the metric
    refine_ms = event_ms(lambda: ifmm.solve(fact, b_dev, refine=4, target=10 * tol), reps=1)
    refine_hist = list(fact.last_refinement)
    r_m, top_dim, shard = fact.r_m, fact.top_dim, fact.shard
    # free the last factorization first so later ones reuse its device slabs
    del fact

    # e2e through the public API with host buffers (H2D of b, D2H of x inside)
    e2e_times = []
    for _ in range(max(1, min(args.steps, 2))):
        torch.cuda.synchronize()
        ta = time.perf_counter()
        f2 = factor()
        ifmm.solve(f2, b_host)
        e2e_times.append(time.perf_counter() - ta)
        del f2
    e2e = float(np.mean(e2e_times))
    if ws > 1:
        te = torch.tensor([e2e], device=red_dev)
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = float(te.item())

    # instrumented factorization: per-phase device time (CUDA events on the library stream)
    ft = factor(timing=True)
    ph = ft.phase_times
    work = ft.work
    work_all = dict(work)
    if ws > 1:  # per-rank work -> whole job
        keys = ("flops_exec", "flops_schur", "flops_ref", "solve_bytes", "flops_lu", "flops_x")
        wt = torch.tensor([work[k] for k in keys], dtype=torch.float64, device=red_dev)
        dist.all_reduce(wt)
        work_all = dict(zip(keys, wt.tolist()))
    fl_peak = measured_fp64_peak()
    hb, hb_src = hbm_peak()
    fac_ms_dev = sum(v[0] for v in ph.values())

    def tensor_phase(name, flops):
        ms, nl = ph[name]
        a = flops / (ms * 1e-3) / 1e12 if ms > 0 else None
        return {"ms": round(ms, 3), "launches": nl, "flops": flops, "achieved": a, "peak": fl_peak,
                "unit": "TFLOP/s", "frac": a / fl_peak if a else None, "bound": "tensor"}

    phases = {
        "lu": tensor_phase("lu", work["flops_lu"]),
        "x_solve": tensor_phase("x_solve", work["flops_x"]),
        "schur": tensor_phase("schur", work["flops_schur"]),
        "compress": {"ms": round(ph["compress"][0], 3), "launches": ph["compress"][1], "bound": "latency",
                     "note": "ACA + recompression + basis augmentation of small fills: no flop/byte roofline"},
        "gather": {"ms": round(ph["gather"][0], 3), "launches": ph["gather"][1], "bound": "hbm"},
        "transition": {"ms": round(ph["transition"][0], 3), "launches": ph["transition"][1], "bound": "hbm"},
        "top": tensor_phase("top", 0.0) | {"note": "level-2 LU, counted in lu flops"},
    }
    # dominant kernel for the roofline line: the phase with the most device time among the tensor phases
    dom = max(("lu", "x_solve", "schur"), key=lambda k: phases[k]["ms"])
    dom_kernel = {"lu": "lu_panel/lu_swap_trsm/lu_update (batched getrf)",
                  "x_solve": "lu_xsolve_kernel (X = S^-1 C, blocked triangular solves on DMMA)",
                  "schur": "schur_concat_kernel (Schur update T = C^T X, DMMA)"}[dom]

    # solve: HBM roofline (the records are streamed once per sweep)
    solve_ms = event_ms(lambda: ifmm.solve(ft, b_dev))
    b32 = torch.from_numpy(np.random.default_rng([0, 2]).standard_normal((N, 32))).cuda()
    ifmm.solve(ft, b32)
    solve32_ms = event_ms(lambda: ifmm.solve(ft, b32))
    solve32_flops = 2.0 * work["solve_bytes"] / 8.0 * 32
    # matvec: HBM roofline (every stored operator block read once)
    nb = store.nbytes
    mv_bytes = nb["p2p"] + nb["m2l"] + 2 * nb["basis"]
    mv_ms = event_ms(lambda: ifmm.fmm_matvec(store, tree, b_dev))
    asm_bytes = nb["p2p"] + nb["m2l"] + nb["basis"]

    def hbm(bytes_, ms):
        a = bytes_ / (ms * 1e-3) / 1e9
        return {"ms": round(ms, 3), "bytes": bytes_, "achieved": a, "peak": hb, "unit": "GB/s", "frac": a / hb,
                "peak_source": hb_src}

    # extension: the same step with rank-growth control at eps / 10
    rank_control = None
    phase_by_level = ft.phase_times_by_level
    shard_comm_ms = ft.shard["comm_ms"] if ws > 1 else None
    if rt_main is not None:
        rank_control = {"rank_tol": rt_main, "rank_sum_before_after": list(ft.rank_control),
                        "note": "measured with rank-growth control (extension, csrc/consolidate.cu; C5_4m / C5 only "
                                "fit in HBM with it): `value` and every other number of this line use it"}
    elif ws == 1:
        del ft
        rt = tol / 10.0
        rc_times, frc, xrc = [], None, None
        for it in range(1 + max(1, min(args.steps, 3))):  # one warm-up
            if frc is not None:
                del frc
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            frc = ifmm.factorize(store, tree, pivot_condition_limit=PIVOT_LIMIT, on_singular="record", rank_tol=rt)
            xrc = ifmm.solve(frc, b_dev)
            e1.record()
            torch.cuda.synchronize()
            if it > 0:
                rc_times.append(e0.elapsed_time(e1) / 1e3)
        rr = ifmm.fmm_matvec(store, tree, xrc.double()) - b_dev
        ifmm.solve(frc, b_dev, refine=1)
        rank_control = {
            "rank_tol": rt, "value": float(np.mean(rc_times)), "unit": "s",
            "relative_residual": float(torch.linalg.norm(rr) / torch.linalg.norm(b_dev)),
            "residual_after_one_refinement_step": frc.last_refinement[-1],
            "rank_sum_before_after": list(frc.rank_control), "top_dim": frc.top_dim, "r_m": frc.r_m,
            "pivots_over_limit": len(frc.singular_pivots), "flops_exec": frc.work["flops_exec"],
            "note": "extension, not in value: every pivot's coupling row (its M2L blocks + its rows of the parent's "
                    "basis) re-truncated at rank_tol right before its elimination (csrc/consolidate.cu); the "
                    "reference never calls its _maybe_consolidate, so `value` stays the parity path"}
        del frc

    ref_c3 = None
    if args.config == "C3":
        g = np.load(os.path.join(ROOT, "tests", "golden", "c3_1m.npz"))
        ref_c3 = {"morton": int(len(g["singular_morton"])), "colour9": int(len(g["singular_colour9"])),
                  "resid_morton": float(g["resid_morton"]), "resid_colour9": float(g["resid_colour9"])}
    # DRAM traffic of one launch of the dominant kernel from the committed ncu --set full capture
    traffic = {}
    tp = os.path.join(ROOT, "profiles", {"x_solve": "r02_xsolve_l5_ncu.json", "schur": "r01_schur_l5_ncu.json"}.get(
        dom, "none.json"))
    if os.path.exists(tp):
        with open(tp) as fh:
            traffic = json.load(fh)
        traffic["source_file"] = os.path.relpath(tp, ROOT)
    line = {
        "metric": METRIC, "value": t_step, "unit": "s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_step * 1e3, "higher_is_better": False, "scaling": "strong" if ws > 1 else "weak",
        "vs_baseline": None,
        "dtype": "f64", "data": ("synthetic (seeded 16-component Gaussian mixture in [0,1]^2, std 0.05, clipped; "
                                 "N(0,1) rhs)" if sparse else
                                 "synthetic (seeded uniform points in [0,1]^2, N(0,1) rhs)"),
        "config": {"workload": args.config, "N": N, "kernel": "1/|x-y|" if kern == "inv_r" else "log|x-y|",
                   "diag": "sqrt(N)", "depth": depth, "p": p, "eps": tol, "nrhs": nrhs,
                   "parallelism": f"subtree{ws} (level-2 subtrees per rank, {args.transport} halo exchange per "
                                  f"colour batch)" if ws > 1 else "single",
                   "pivot_condition_limit": PIVOT_LIMIT, "on_singular": "record", "rank_tol": rt_main,
                   "tree": (f"uniform depth {depth} with empty cells accepted ({int((np.diff(tree.leaf_offsets) == 0).sum())} "
                            f"of {4 ** depth} empty, at most {int(np.diff(tree.leaf_offsets).max())} points in a cell); "
                            "NOT the adaptive tree of BASELINE config 4") if sparse else f"uniform depth {depth}",
                   "l2": "factor state (GBs) >> 126 MB L2; no flush needed"},
        "relative_residual": resid,
        "pivots_over_limit": {"count": len(singular), "first": singular[:4], "max_cond_by_level": max_cond,
                              "reference_counts_at_C3": ref_c3,
                              "note": "the reference raises SingularPivotError at the first such pivot; at C3 it "
                                      "meets them itself, so both sides record and continue"},
        "refined_solve": {"target": 10 * tol, "steps": len(refine_hist) - 1, "residual_history": refine_hist,
                          "ms": refine_ms,
                          "note": "extension: x += solve(b - A~x) with the store's FMM operator; not in value"},
        "r_m": r_m, "top_dim": top_dim,
        "assembly": {"tree_s": t_tree, "operators_s": t_assembly,
                     "roofline": hbm(asm_bytes, t_assembly * 1e3) | {"bytes_note": "operator blocks written "
                                                                                   "once (P2P, M2L, bases); wall "
                                                                                   "clock incl. host planning"}},
        "flops": {"exec": work_all["flops_exec"], "schur": work_all["flops_schur"], "lu": work_all["flops_lu"],
                  "x_solve": work_all["flops_x"], "reference_equiv": work_all["flops_ref"],
                  "fp64_tflops_step": work_all["flops_exec"] / t_step / 1e12,
                  "step_frac_of_peak": work_all["flops_exec"] / t_step / 1e12 / fl_peak,
                  "scope": "whole job (summed over ranks)" if ws > 1 else "one GPU"},
        "shard": {"rank0_halo_bytes_per_factorization": shard["halo_bytes"],
                  "rank0_meta_bytes": shard["meta_bytes"], "exchanges": shard["exchanges"],
                  "rank0_comm_ms": shard_comm_ms} if ws > 1 else None,
        "phases": phases,
        "phase_ms_by_level": phase_by_level,
        "roofline": {"kernel": dom_kernel, "bound": "tensor", "achieved": phases[dom]["achieved"], "peak": fl_peak,
                     "unit": "TFLOP/s", "frac": phases[dom]["frac"], "traffic": traffic.get("dram_bytes_per_launch"),
                     "traffic_launch": traffic.get("kernel"), "traffic_source": traffic.get("source_file"),
                     "launches": phases[dom]["launches"],
                     "share_of_factor": phases[dom]["ms"] / fac_ms_dev if fac_ms_dev else None,
                     "achieved_source": "algorithmic flops of the phase / CUDA-event time of its launches on the "
                                        "library stream (instrumented factorization)",
                     "peak_source": "measured live: cuBLAS DGEMM 8192^3 (torch.matmul float64)"},
        "solve_roofline": hbm(work["solve_bytes"], solve_ms) | {"bound": "hbm"},
        "matvec_roofline": hbm(mv_bytes, mv_ms) | {"bound": "hbm", "bytes_note": "P2P + M2L + 2 x bases"},
        "solve_32rhs": {"ms": solve32_ms, "tflops": solve32_flops / (solve32_ms * 1e-3) / 1e12,
                        "frac_of_fp64_peak": solve32_flops / (solve32_ms * 1e-3) / 1e12 / fl_peak,
                        "vs_32_single_solves": 32 * solve_ms / solve32_ms,
                        "note": "extension (SURVEY 8f item 1): one factorization, 32 rhs as DMMA GEMM sweeps; "
                                "not in value"},
        "rank_control": rank_control,
        "e2e": {"value": e2e, "unit": "s", "h2d_bytes_per_step": 8 * N * nrhs, "d2h_bytes_per_step": 8 * N * nrhs},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        ns, ds = SAMPLE[args.config]
        tf, tsv = oracle_step_seconds(ns, ds, p, tol, kern)
        line["cpu_baseline"] = {"value": tf + tsv, "unit": "s", "cores": 1, "kind": "port",
                                "sample": sample_desc(args.config, ns, ds) + f": factor {tf:.2f} s + solve {tsv:.3f} s"}
        if args.config == "C3":
            line["cpu_baseline"]["c3_full_run"] = c3_full_run()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
