#!/usr/bin/env python
"""Per-kernel device times of one workload, joined with the plan (dev tool).

  python tools/kernel_times.py su2random 28 [key=value options...]
"""
import json
import os
import sys
from collections import Counter

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2408_09055_b200 import atlas as A  # noqa: E402
from workloads import circuits as C  # noqa: E402

fam, n = sys.argv[1], int(sys.argv[2])
opts = {kv.split("=")[0]: int(kv.split("=")[1]) for kv in sys.argv[3:]}
c = C.make(fam, n)
s = A.Simulator(n, 0, 1, 0, **opts)
s.load_circuit(c.gates)
s.plan()
pj = s.plan_json()
s.run()
s.set_option("timing", 1)
reps = 3
rows = None
for _ in range(reps):
    s.run()
    L = [(k, t) for k, t, b in s.launches() if k in ("fused", "shm")]
    rows = L if rows is None else [(k, t0 + t) for (k, t0), (_, t) in zip(rows, L)]
ks = [k for st in pj["stages"] for k in st["kernels"]]
assert len(ks) == len(rows), (len(ks), len(rows))
out = []
for k, (kind, t) in zip(ks, rows):
    kinds = Counter(c.gates[g].kind for g in k["gates"])
    out.append({"kind": k["kind"], "ms": round(t / reps, 4), "phases": k.get("phases"),
                "nq": len(k["qubits"]), "gates": dict(kinds)})
    print(json.dumps(out[-1]))
json.dump(out, open(os.path.join(ROOT, "gpurun_out", f"ktimes_{fam}{n}.json"), "w"))
