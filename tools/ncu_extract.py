"""Extract the roofline-relevant metrics of every launch in an `ncu --page raw --csv` export."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
tag = sys.argv[2]
if len(rows) < 3:
    sys.exit(0)
h, units = rows[0], rows[1]
want = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"]
idx = [h.index(w) if w in h else -1 for w in want]
for r in rows[2:]:
    vals = [(r[i] if i >= 0 else "") for i in idx]
    vals[0] = vals[0].split("(")[0].replace("void ", "").replace("ifmm::", "")
    out = [tag]
    for k, (i, v) in enumerate(zip(idx, vals)):
        u = units[i] if (i >= 0 and k >= 3) else ""
        out.append(v.replace(",", "") + (" " + u if u and u != "%" else ""))
    print(",".join(out))
