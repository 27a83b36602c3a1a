#!/usr/bin/env python
"""Opcode mix of one kernel from `ncu -i X --page source --csv --print-source sass`:
warp instructions executed per opcode, per unit (argv[2] = warps x tiles)."""
import csv
import sys
from collections import Counter

path = sys.argv[1]
div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
rows = list(csv.reader(open(path)))
h = rows[1]
ie = h.index("Instructions Executed")
src = h.index("Source")
stall = h.index("Warp Stall Sampling (All Samples)")
c, s = Counter(), Counter()
for r in rows[2:]:
    if len(r) <= ie:
        continue
    op = r[src].strip().split()
    if not op:
        continue
    o = op[0]
    if o.startswith("@"):
        o = op[1]
    o = o.split(".")[0]
    try:
        c[o] += float(r[ie]); s[o] += float(r[stall] or 0)
    except ValueError:
        pass
tot = sum(c.values()); st = sum(s.values())
print(f"total {tot / div:.1f} per unit")
for o, n in c.most_common(25):
    print(f"{o:10s} {n / div:9.1f}  {100 * n / tot:5.1f}%  stall-samples {100 * s[o] / max(st, 1):5.1f}%")
