"""Per-kernel totals of an `ncu --metrics gpu__time_duration.sum --csv` launch list."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[i]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[i + 1:]:
    if len(r) > vi:
        n = r[ki].split("(")[0].replace("void ", "")
        n = re.sub(r"ifmm::\(anonymous namespace\)::|ifmm::<unnamed>::|ifmm::", "", n)
        agg[n][0] += 1
        agg[n][1] += float(r[vi].replace(",", ""))
tot = sum(v[1] for v in agg.values())
print(f"total {sum(v[0] for v in agg.values())} launches, {tot / 1e6:.2f} ms (ncu serialised, cold)")
for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{n[:58]:58s} {c:6d} {t / 1e6:9.2f} ms {100 * t / tot:5.1f}%")
