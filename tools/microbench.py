#!/usr/bin/env python
"""Kernel microbenchmarks through the C-ABI (dev tool, GPU only).

Builds small circuits that lower to exactly one kernel of a chosen shape on
an n-qubit shard and reports the per-launch CUDA-event time and HBM GB/s
(algorithmic bytes 2 * 2^n * 16 per pass).

  python tools/microbench.py [--n 28] [--reps 5]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2408_09055_b200 import atlas as A  # noqa: E402
from workloads.circuits import Gate  # noqa: E402


def timed(n, gates, reps, dtype=0, **opt):
    s = A.Simulator(n, dtype, 1, 0, **opt)
    s.load_circuit(gates)
    s.plan(4, 3.0)
    st = s.plan_stats()
    pj = s.plan_json()
    for _ in range(2):
        s.run()
    s.set_option("timing", 1)
    rows = []
    for _ in range(reps):
        s.run()
        rows += [(k, t, b) for k, t, b in s.launches() if k in ("fused", "shm")]
    s.close()
    ks = [k for stg in pj["stages"] for k in stg["kernels"]]
    t = sorted(r[1] for r in rows)
    med = t[len(t) // 2]
    byts = rows[0][2]
    return {"kernels": [(k["kind"], len(k["gates"]), k.get("phases")) for k in ks],
            "ms": round(med, 4), "GBps": round(byts / med / 1e6, 1),
            "launches_per_run": len(rows) // reps}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=28)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    n = a.n
    out = []

    def rec(name, gates, **opt):
        try:
            r = timed(n, gates, a.reps, **opt)
        except Exception as e:  # noqa: BLE001
            r = {"error": str(e)}
        r["name"] = name
        out.append(r)
        print(json.dumps(r), flush=True)

    # fused kernels k = 1..5 on high and low qubits
    for k in range(1, 6):
        for where, qs in (("low", list(range(5, 5 + k))), ("high", list(range(n - k, n)))):
            g = [Gate("H", (q,)) for q in qs] + [Gate("RX", (q,), (0.3,)) for q in qs]
            rec(f"fused k={k} {where}", g, kinds=1, kernelizer=1)
    # near-empty shared-memory kernels (CX chains are folded into addresses)
    for K in (10, 11, 12):
        for where, qs in (("contig", list(range(5, K))), ("high", list(range(n - (K - 5), n))),
                          ("spread", [5 + i * ((n - 6) // (K - 5)) for i in range(K - 5)])):
            g = [Gate("CX", (qs[i], qs[i + 1])) for i in range(len(qs) - 1)]
            for nb in (1, 2):
                rec(f"shm-empty K={K} {where} nbuf={nb}", g, kinds=2, kernelizer=1, shm_qubits=K,
                    shm_nbuf=nb)
    # shared-memory kernels with dense work: H on every active qubit
    for K in (12,):
        qs = list(range(n - (K - 5), n))
        for reps in (1, 2, 4):
            g = []
            for _ in range(reps):
                g += [Gate("H", (q,)) for q in list(range(5)) + qs]
            rec(f"shm-H x{reps} K={K} high", g, kinds=2, kernelizer=1, shm_qubits=K)
        # diagonal-heavy: all CP pairs (qft-like)
        g = [Gate("H", (q,)) for q in qs] + [Gate("CP", (qs[i], qs[j]), (0.1 * (i + j),))
                                              for i in range(len(qs)) for j in range(i + 1, len(qs))]
        g += [Gate("CP", (i, qs[j]), (0.2,)) for i in range(5) for j in range(len(qs))]
        rec(f"shm-CP K={K} high", g, kinds=2, kernelizer=1, shm_qubits=K)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "microbench.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
