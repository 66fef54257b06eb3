# ncu --set full of one kernel (regex $1, skip $2) of the C3 step; prints the stall breakdown
ncu -f --set full --clock-control none -k "regex:$1" -s "${2:-0}" -c 1 -o /tmp/k_st python tools/profile_step.py C3 > /dev/null 2>&1
ncu -i /tmp/k_st.ncu-rep --page raw --csv > /tmp/k_st.csv 2>/dev/null
python - <<'PY'
import csv
r = list(csv.reader(open('/tmp/k_st.csv'))); h = r[0]; v = r[2]
def f(x):
    try: return float(x.replace(',', ''))
    except ValueError: return 0.0
items = sorted([(k, f(v[i])) for i, k in enumerate(h) if 'average_warps_issue_stalled' in k and k.endswith('per_issue_active.ratio')], key=lambda x: -x[1])
for k, x in items[:10]: print(f"  {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):28s} {x:.2f}")
for k in ['sm__inst_executed.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active', 'gpu__time_duration.sum', 'sm__warps_active.avg.pct_of_peak_sustained_active']:
    print(' ', k, v[h.index(k)] if k in h else '?')
PY
