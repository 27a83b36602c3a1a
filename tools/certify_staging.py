#!/usr/bin/env python
"""Certify the staging optimum of every BASELINE.json multi-GPU config with
the paper's own method: the staging ILP (objective Eq. P:L1491, constraints
P:L1495-1502) solved by an off-the-shelf ILP solver (HiGHS via scipy; the
paper used PuLP + HiGHS), for s = 1, 2, ... until feasible (Alg.
Stage P:L1525-1533, Thm. ilp-optimal).  Calls only oracle/ (test
infrastructure); writes tests/golden/staging_ilp_bj.json, which
tests/test_planner_scale.py compares the product planner against.

    python tools/certify_staging.py [--quick]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import planner as P  # noqa: E402
from workloads import circuits as C  # noqa: E402

CONFIGS = [("qft", 32, 4), ("ising", 32, 4)] + \
    [(f, 33, W) for f in ("qft", "ghz", "graphstate", "qsvm", "wstate", "su2random") for W in (2, 4, 8)] + \
    [("qft", 35, 8), ("su2random", 35, 8), ("qft", 36, 8), ("su2random", 36, 8)]
COST_C = 3.0


def main():
    out = {"_source": "tools/certify_staging.py: oracle.planner.ilp_highs (the staging ILP of "
                      "P:L1491-1502 solved by HiGHS), s = 1, 2, ... until feasible; c = 3 "
                      "(P:L1975); R = 0 (L = n - log2 W local, G = log2 W global qubits)",
           "configs": []}
    for fam, n, W in CONFIGS:
        G = {2: 1, 4: 2, 8: 3}[W]
        L = n - G
        c = C.make(fam, n)
        facts = P.gate_facts(c)
        t0 = time.time()
        rec = {"family": fam, "n": n, "world": W, "L": L, "G": G, "c": COST_C, "infeasible_s": []}
        for s in range(1, 9):
            obj, opt, locs = P.ilp_highs(c, L, G, s, COST_C, facts=facts, time_limit=900)
            if obj is None:
                assert opt, f"{fam} n={n} W={W} s={s}: solver stopped without a proof"
                rec["infeasible_s"].append(s)
                continue
            assert opt, f"{fam} n={n} W={W} s={s}: not proven optimal"
            rec["s"] = s
            rec["cost"] = obj
            break
        rec["solve_s"] = round(time.time() - t0, 1)
        print(json.dumps(rec), flush=True)
        out["configs"].append(rec)
    path = os.path.join(ROOT, "tests", "golden", "staging_ilp_bj.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
