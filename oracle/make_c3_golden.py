"""Pack the two oracle/run_c3.py outputs (GPU-box host run) into tests/golden/c3_1m.npz
and profiles/r02_c3_reference_cpu.json.  TEST INFRASTRUCTURE ONLY.

    python oracle/make_c3_golden.py gpurun_out/c3
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    src = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "c3")
    out = {}
    summ = {}
    for order in ("morton", "colour9"):
        g = np.load(f"{src}_{order}.npz")
        with open(f"{src}_{order}.json") as f:
            summ[order] = json.load(f)
        if order == "morton":
            out["perm"] = g["perm"].astype(np.int32)
            out["leaf_off"] = g["leaf_off"].astype(np.int64)
        else:
            assert np.array_equal(out["perm"], g["perm"]), "the two runs built different trees"
        out[f"x_{order}"] = g["x"]
        out[f"resid_{order}"] = g["resid"]
        out[f"top_{order}"] = g["top"]
        out[f"rm_{order}"] = g["r_m"]
        out[f"stats_{order}"] = g["stats"]
        out[f"singular_{order}"] = g["singular"]
        out[f"max_cond_{order}"] = g["max_cond"]
        out[f"rank_sum_{order}"] = g["rank_sum"]
    out.update(N=1048576, depth=7, p=4, tol=1e-6, kernel="inv_r", a=0.001, seed=0)
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "c3_1m.npz"), **out)
    keep = ("t_tree", "t_a", "t_f", "t_s", "t_s_all", "level_done_s", "top", "r_m", "resid", "singular_count",
            "first_singular", "max_cond", "peak_rss_gb", "cores_used", "host_cpus", "blas_threads")
    rep = {
        "what": "CPU oracle (bit-exact restatement of the reference, oracle/ifmm_oracle.py) at BASELINE C3 "
                "itself, run on the GPU box's host by oracle/run_c3.py (tools/c3_oracle_job.sh), one process "
                "per elimination order, each pinned to one core with one BLAS thread",
        "config": "N=1,048,576 uniform [0,1]^2 seed 0, K=1/|x-y| diag sqrt(N), depth 7, p=4, eps=1e-6, 1 N(0,1) rhs",
        "reference_semantics": "the reference raises SingularPivotError at the first pivot whose dgecon estimate "
                               "exceeds 1e12 (ifmm/solver.py:50,214-218); the run records such pivots and goes on",
        **{o: {k: summ[o][k] for k in keep} for o in summ},
    }
    with open(os.path.join(ROOT, "profiles", "r02_c3_reference_cpu.json"), "w") as f:
        json.dump(rep, f, indent=1)
    print(json.dumps({o: (summ[o]["t_f"], summ[o]["resid"], summ[o]["first_singular"]) for o in summ}))


if __name__ == "__main__":
    main()
