"""Per-level kernel times of the C3 step from an ncu launch list (csv or csv.gz).
    python tools/level_kernels.py launches.csv[.gz] [TOP]
Batches are delimited by lu_perm_init launches (9 colour batches per level)."""
import collections
import csv
import gzip
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 14
txt = (gzip.open(path, "rt") if path.endswith(".gz") else open(path)).read()
lines = txt.splitlines()
hi = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rd = list(csv.reader(lines[hi:]))
h, rows = rd[0], rd[1:]
ni, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
batch = -1
per = collections.defaultdict(lambda: collections.defaultdict(lambda: [0, 0.0]))
for r in rows:
    if len(r) <= vi:
        continue
    name = r[ni].split("(")[0].replace("void ", "").replace("ifmm::", "").replace("<unnamed>::", "")
    if name.startswith("lu_perm_init"):
        batch += 1
    if batch < 0:
        continue
    lvl = 7 - batch // 9 if batch < 54 else 1
    t = float(r[vi].replace(",", ""))
    t = t / 1e3 if r[ui] == "ns" else t * 1e3 if r[ui] == "ms" else t
    per[lvl][name][0] += 1
    per[lvl][name][1] += t
for lvl in sorted(per, reverse=True):
    tot = sum(v[1] for v in per[lvl].values())
    print(f"level {lvl}: {tot / 1e3:.1f} ms")
    for n, (c, t) in sorted(per[lvl].items(), key=lambda x: -x[1][1])[:top]:
        print(f"   {n[:50]:50s} {c:5d} {t / 1e3:8.2f} ms")
