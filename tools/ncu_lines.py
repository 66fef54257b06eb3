"""Hottest CUDA source lines of an ncu report (warp-stall samples, instructions).
    python tools/ncu_lines.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, fname = [], None
for line in out.splitlines():
    if line.startswith('"File Path"'):
        fname = line.split('","')[1].rstrip('"').split("/")[-1]
        continue
    if line.startswith('"Function Name"') or line.startswith('"Line No"'):
        continue
    r = next(csv.reader(io.StringIO(line)))
    if len(r) > 7 and r[2] == "-":  # a source line row (not a SASS row)
        rows.append((fname, r[0], r[1], float(r[4] or 0), float(r[7] or 0)))
ts = sum(x[3] for x in rows) or 1
ti = sum(x[4] for x in rows) or 1
for f, ln, src, s, i in sorted(rows, key=lambda x: -x[3])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{100 * s / ts:5.1f}% stall {100 * i / ti:5.1f}% inst  {f}:{ln}  {src.strip()[:90]}")
