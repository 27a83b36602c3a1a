"""Summarise an ncu source page (cuda,sass) by CUDA source line: instructions
executed and warp-stall samples.  Dev tool: python tools_ncu_source.py rep.ncu-rep"""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"][0]
h = rows[hi]
ie = h.index("Instructions Executed")
ss = h.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, k in enumerate(h) if k.startswith("stall_")]
src = {}
agg = defaultdict(lambda: [0, 0])
stalls = defaultdict(float)
cur = None
for r in rows[hi + 1:]:
    if not r:
        continue
    if r[0] in ("File Path", "Function Name", "Line No"):
        continue
    if r[0]:  # a CUDA source line
        try:
            cur = int(r[0])
        except ValueError:
            continue
        src[cur] = r[1]
    def f(x):
        try:
            return float(x.replace(",", ""))
        except Exception:
            return 0.0
    if len(r) > ie and r[2]:
        agg[cur][0] += f(r[ie])
        agg[cur][1] += f(r[ss])
        for c in stall_cols:
            stalls[h[c]] += f(r[c])
tot_i = sum(v[0] for v in agg.values()) or 1
tot_s = sum(v[1] for v in agg.values()) or 1
print(f"total warp instructions {tot_i:.3e}, stall samples {tot_s:.0f}")
for ln, (i, s) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{ln:5d} inst {100*i/tot_i:5.1f}%  stall {100*s/tot_s:5.1f}%  {src.get(ln,'')[:90]}")
print("stall reasons:", ", ".join(f"{k[6:]}={100*v/max(sum(stalls.values()),1):.0f}%" for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:8]))
