# ncu --set full capture of one launch of a kernel in the C3 step (regex $1, skip $2, tag $3);
# keeps the report in gpurun_out/ and prints the stall breakdown + headline metrics.
# usage (on the GPU box): bash tools/ncu_capture.sh lu_xsolve 18 xsolve_l5 [CONFIG [rank_tol]]
cfg=${4:-C3}
ncu -f --set full --import-source on --clock-control none -k "regex:$1" -s "${2:-0}" -c 1 \
    -o gpurun_out/ncu_$3 python tools/profile_step.py $cfg $5 > /dev/null 2>&1
ncu -i gpurun_out/ncu_$3.ncu-rep --page raw --csv > /tmp/k_$3.csv 2>/dev/null
python - /tmp/k_$3.csv $3 <<'PY'
import csv, sys
r = list(csv.reader(open(sys.argv[1]))); h = r[0]; u = r[1]; v = r[2]
def f(x):
    try: return float(x.replace(',', ''))
    except ValueError: return 0.0
print("==", sys.argv[2], v[h.index("Kernel Name")][:80], "grid", v[h.index("Grid Size")], "block", v[h.index("Block Size")])
for k in ['gpu__time_duration.sum', 'sm__warps_active.avg.pct_of_peak_sustained_active',
          'smsp__issue_active.avg.pct_of_peak_sustained_active',
          'sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active',
          'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
          'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
          'lts__t_sector_hit_rate.pct', 'launch__registers_per_thread', 'launch__occupancy_limit_shared_mem']:
    print(f"  {k:80s} {v[h.index(k)] if k in h else '?'} {u[h.index(k)] if k in h else ''}")
items = sorted([(k, f(v[i])) for i, k in enumerate(h) if 'average_warps_issue_stalled' in k and k.endswith('per_issue_active.ratio')], key=lambda x: -x[1])
for k, x in items[:8]: print(f"  stall {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):28s} {x:.2f}")
PY
