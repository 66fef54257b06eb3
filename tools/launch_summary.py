"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hdr_i]; ki = h.index('Kernel Name'); vi = h.index('Metric Value')
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for r in rows[hdr_i + 1:]:
    if len(r) <= vi: continue
    name = r[ki].split('(')[0].replace('void ', '').replace('ifmm::', '')
    try: v = float(r[vi].replace(',', ''))
    except ValueError: continue
    a = agg[name]; a[0] += 1; a[1] += v; a[2] = max(a[2], v)
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f"{k[:60]:60s} n={v[0]:5d} total={v[1]/1e6:9.2f} ms  max={v[2]/1e6:8.2f} ms share={v[1]/tot:6.1%}")
print(f"total {tot/1e6:.2f} ms")
