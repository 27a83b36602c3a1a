#!/usr/bin/env python
"""K04: calibrate the Kernelize cost model on a B200 with OUR kernels.

PAPER.md P:L1995-1997: "For fusion kernels, we measure their execution time
with different numbers of qubits.  For shared-memory kernels, we measure the
run time of an empty shared-memory kernel to estimate the cost of loading a
state vector to GPU shared memory, and profile the run times for different
types of gates using the GPU shared memory."

Units (R11): integer nanoseconds per 2^28-amplitude shard, i.e.
the device time of one launch at n = 28 (fp64 and fp32 both measured at
n = 28).  Writes gpurun_out/costmodel_b200_<dtype>.json (SPEC S:L358 format)
(copied to profiles/ by hand) and prints it.

  python tools/calibrate.py [--dtype c128|c64] [--reps 5]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2408_09055_b200 import atlas as A  # noqa: E402
from workloads.circuits import ARITY, NPARAMS, Gate  # noqa: E402

N = 28


def launch_ms(gates, dtype, reps, **opt):
    # init_fuse=0: the measured launch must read and write the shard (the
    # fused |0> initialisation would make the first kernel write-only);
    # ls_qubits fixed so the calibration circuits keep their one-kernel plans
    opt.setdefault("ls_qubits", 5)
    s = A.Simulator(N, dtype, 1, 0, kernelizer=1, init_fuse=0, **opt)
    s.load_circuit(gates)
    s.plan(4, 3.0)
    pj = s.plan_json()
    nk = sum(len(st["kernels"]) for st in pj["stages"])
    s.run()
    s.set_option("timing", 1)
    t = []
    for _ in range(reps):
        s.run()
        t += [ms for k, ms, b in s.launches() if k in ("fused", "shm")]
    s.close()
    return statistics.median(t), nk


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dtype", default="c128", choices=["c128", "c64"])
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    dt = 0 if a.dtype == "c128" else 1
    K = 12 if dt == 0 else 13
    ns = lambda ms: int(round(ms * 1e6))  # noqa: E731
    high = list(range(N - (K - 5), N))   # the active non-LSB qubits of a tile
    act = list(range(5)) + high
    # fusion kernels by qubit count, averaged over a low and a high placement
    fusion = []
    for q in range(1, 6):
        v = []
        for qs in (list(range(5, 5 + q)), list(range(N - q, N))):
            g = [Gate("H", (x,)) for x in qs] + [Gate("RX", (x,), (0.3,)) for x in qs]
            ms, nk = launch_ms(g, dt, a.reps, kinds=1)
            assert nk == 1
            v.append(ms)
        fusion.append(ns(statistics.mean(v)))
        print("fusion", q, fusion[-1], flush=True)
    # alpha: the empty shared-memory kernel (one identity-like diagonal gate)
    alpha_ms, nk = launch_ms([Gate("Z", (high[0],))], dt, a.reps, kinds=2, shm_qubits=K)
    assert nk == 1
    alpha = ns(alpha_ms)
    print("alpha", alpha, flush=True)
    # per-gate marginal cost inside a shared-memory kernel
    import numpy as np
    rng = np.random.default_rng(7)
    M = 48
    gate_cost = {}
    for kind in ARITY:
        k = ARITY[kind]
        g = []
        for i in range(M):
            qs = tuple(int(x) for x in rng.choice(act, size=k, replace=False))
            ps = tuple(float(x) for x in rng.uniform(0, 6.28, size=NPARAMS[kind]))
            g.append(Gate(kind, qs, ps))
        ms, nk = launch_ms(g, dt, a.reps, kinds=2, shm_qubits=K)
        assert nk == 1, (kind, nk)
        gate_cost[kind] = max(0, ns((ms - alpha_ms) / M))
        print("gate", kind, gate_cost[kind], flush=True)
    model = {"fusion_cost": fusion, "alpha": alpha, "gate_cost": gate_cost,
             "q_max_fusion": 5, "q_max_shared": K, "ls_qubits": 5,
             "_source": f"calibrated-b200-{a.dtype}"}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    out = os.path.join(ROOT, "gpurun_out", f"costmodel_b200_{a.dtype}.json")
    json.dump(model, open(out, "w"), indent=1)
    print(json.dumps(model))


if __name__ == "__main__":
    main()
