#!/usr/bin/env python
"""Summarise ncu output for profiles/ (run here, on the CPU box).

  python tools/ncu_summary.py launches <launches.csv>            -> per-kernel share table
  python tools/ncu_summary.py full <prof.ncu-rep> [<key>]        -> key metrics per launch
  python tools/ncu_summary.py traffic <prof.ncu-rep> <key>       -> update profiles/traffic.json

`key` names the bench line the capture belongs to (e.g. shm_su2random_n28_f64);
bench.py reads profiles/traffic.json[key] for roofline.traffic (bytes per launch).
"""
from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

FULL_METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__shared_mem_per_block_dynamic",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "sm__cycles_elapsed.avg.per_second",
]


def launches(path):
    """Per-kernel share table; the plan-specialised SHM kernels (one
    atlas_shm_<hash> per launch of the plan) are also summed as one row."""
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
    for r in rows[1:]:
        if r[h.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        k = r[ki].split("(")[0]
        agg[k][0] += 1
        agg[k][1] += float(r[vi].replace(",", "")) * scale[r[ui]]
    tot = sum(v[1] for v in agg.values())
    jit = [v for k, v in agg.items() if k.startswith("atlas_shm_")]
    if jit:
        agg["ALL atlas_shm_* (plan-specialised SHM kernels)"] = [sum(v[0] for v in jit),
                                                                 sum(v[1] for v in jit)]
    out = ["| kernel | launches | total ms | avg ms | share |", "|---|---|---|---|---|"]
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{k}` | {c} | {t:.2f} | {t / c:.4f} | {t / tot:.3f} |")
    return "\n".join(out)


def _raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    return rows[0], rows[1], rows[2:]


def full(rep):
    h, u, rows = _raw(rep)
    out = []
    for r in rows:
        out.append(f"### `{r[h.index('Kernel Name')].split('(')[0]}`")
        for m in FULL_METRICS:
            if m in h:
                i = h.index(m)
                out.append(f"- {m} = {r[i]} {u[i]}")
        out.append("")
    return "\n".join(out)


def traffic(rep, key):
    h, u, rows = _raw(rep)
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    vals = []
    for r in rows:
        b = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = h.index(m)
            b += float(r[i].replace(",", "")) * mult[u[i]]
        vals.append(b)
    p = os.path.join(ROOT, "profiles", "traffic.json")
    d = json.load(open(p)) if os.path.exists(p) else {}
    d[key] = int(sum(vals) / len(vals))
    json.dump(d, open(p, "w"), indent=1, sort_keys=True)
    return d[key]


if __name__ == "__main__":
    cmd = sys.argv[1]
    if cmd == "launches":
        print(launches(sys.argv[2]))
    elif cmd == "full":
        print(full(sys.argv[2]))
    elif cmd == "traffic":
        print(traffic(sys.argv[2], sys.argv[3]))
