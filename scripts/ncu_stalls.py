#!/usr/bin/env python
"""Stall-reason totals and top stalled SASS lines of an ncu report: python scripts/ncu_stalls.py rep.ncu-rep"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h = rows[1]
data = rows[2:]
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = {c: 0.0 for c in cols}
si = h.index("Source")
lines = []
for r in data:
    if len(r) < len(h):
        continue
    s = 0.0
    for c in cols:
        try:
            v = float(r[h.index(c)] or 0)
        except ValueError:
            v = 0
        tot[c] += v
        s += v
    lines.append((s, r[si]))
T = sum(tot.values()) or 1
for c, v in sorted(tot.items(), key=lambda kv: -kv[1])[:10]:
    print(f"{c:28s} {100 * v / T:5.1f}%")
print("--- top lines")
for s, l in sorted(lines, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 12]:
    print(f"{100 * s / T:5.1f}%  {l[:110]}")
