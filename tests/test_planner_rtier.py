"""Staging with regional qubits (R > 0) and the staging baseline (NEXT-2).

* R > 0 (option ``regional``): the product's exact staging against the
  oracle's brute force (P:L1474-1516 with L local, R regional, G global
  qubits; objective Eq. P:L1491) on small instances and against the ILP
  solved by HiGHS on medium ones.  Equal-cost optima are not unique, so the
  stage count and the objective are compared, and the product's plan is
  checked to be feasible with exactly the reported objective.
* the SnuQS greedy staging (option ``stager`` = 1): never
  fewer stages than the exact staging (Thm. ilp-optimal);
  the exact staging is monotone in L, and so is it at every L the
  E5 experiment visits.
"""
import pytest

from oracle import planner as P
from workloads import circuits as C

A = pytest.importorskip("paper_2408_09055_b200.atlas")


def product(c, world, cf=3.0, s_max=6, **opt):
    with A.Simulator(c.n, 0, world, 0, kinds=1, kernelizer=2, **opt) as s:
        s.load_circuit(c.gates)
        s.plan(s_max, cf)
        return s.plan_json(), s.plan_stats()


def replay(c, pj, L, cf):
    """Maximal execution of the product's stage sets (oracle side) and the
    objective recomputed by Eq. P:L1477."""
    facts = P.gate_facts(c)
    preds = [[] for _ in facts]
    for a, b in P.dependencies(facts):
        preds[b].append(a)
    done = [False] * len(facts)
    locs, globs = [], []
    for st in pj["stages"]:
        loc = frozenset(st["local"])
        assert len(loc) == L
        done = P.maximal_execution(facts, preds, done, loc)
        locs.append(loc)
        globs.append(frozenset(st["global"]))
    assert all(done)
    return P.stage_cost(locs, globs, cf)


@pytest.mark.parametrize("seed", range(10))
@pytest.mark.parametrize("W,R", [(4, 1), (8, 1), (8, 2)])
def test_regional_staging_matches_bruteforce(seed, W, R):
    n = 6
    c = C.random_circuit(n, 10, 300 + seed, max_arity=2)
    G = W.bit_length() - 1
    L = n - G
    for cf in (0.5, 3.0, 8.0):
        pj, st = product(c, W, cf, s_max=4, regional=R)
        assert st["staging_exact"] == 1
        bf = P.stage_bruteforce(c, L=L, Gq=G - R, s_max=4, c=cf)
        assert pj["staging"]["s"] == bf.s
        assert pj["staging"]["cost"] == pytest.approx(bf.cost)
        assert replay(c, pj, L, cf) == pytest.approx(bf.cost)
        for stg in pj["stages"]:
            assert len(stg["global"]) == G - R and len(stg["regional"]) == R


@pytest.mark.parametrize("fam,n,W,R", [("su2random", 12, 8, 2), ("qft", 13, 16, 2), ("ising", 12, 8, 1),
                                       ("random", 10, 16, 3)])
def test_regional_staging_matches_highs(fam, n, W, R):
    c = C.random_circuit(n, 36, 77, max_arity=2) if fam == "random" else C.make(fam, n)
    G = W.bit_length() - 1
    L = n - G
    pj, st = product(c, W, 2.0, s_max=8, regional=R)
    assert st["staging_exact"] == 1
    facts = P.gate_facts(c)
    for s in range(1, pj["staging"]["s"]):
        obj, proven, _ = P.ilp_highs(c, L, G - R, s, 2.0, facts=facts)
        assert obj is None and proven
    obj, proven, _ = P.ilp_highs(c, L, G - R, pj["staging"]["s"], 2.0, facts=facts)
    assert proven and obj == pytest.approx(pj["staging"]["cost"])
    assert replay(c, pj, L, 2.0) == pytest.approx(obj)


@pytest.mark.parametrize("fam", ["qft", "ising", "su2random", "qsvm", "wstate", "graphstate", "ghz", "random"])
@pytest.mark.parametrize("n,W", [(12, 4), (14, 16), (16, 64)])
def test_greedy_never_beats_exact(fam, n, W):
    """Thm. ilp-optimal: the exact staging has the minimum number of stages,
    so the SnuQS heuristic (E5 baseline) never uses fewer."""
    c = C.random_circuit(n, 3 * n, 5, max_arity=2) if fam == "random" else C.make(fam, n)
    ex, _ = product(c, W, s_max=16)
    gr, gst = product(c, W, s_max=64, stager=1)
    assert gst["staging_exact"] == 0
    assert ex["staging"]["s"] <= gr["staging"]["s"]
    L = n - (W.bit_length() - 1)
    replay(c, gr, L, 3.0)  # the greedy plan is feasible too


@pytest.mark.parametrize("fam", ["qft", "su2random", "random"])
def test_exact_stages_monotone_in_L(fam):
    """more local qubits never need more stages."""
    n = 14
    c = C.random_circuit(n, 40, 9, max_arity=2) if fam == "random" else C.make(fam, n)
    prev = None
    for W in (64, 32, 16, 8, 4, 2):
        pj, _ = product(c, W, s_max=16)
        if prev is not None:
            assert pj["staging"]["s"] <= prev
        prev = pj["staging"]["s"]


def test_regional_c_changes_only_the_objective_on_benchmarks():
    """With R > 0 the objective is S + c T; on the benchmark families every
    remap updates every non-local and every global qubit, so the optimum is
    c-invariant and its objective affine in c (profiles/r02_planner_experiments.md)."""
    c = C.su2random(14)
    plans = []
    for cf in (0.25, 3.0, 10.0):
        pj, st = product(c, 8, cf, s_max=8, regional=2)
        plans.append([(s["local"], s["global"]) for s in pj["stages"]])
        S = sum(len(set(pj["stages"][k]["local"]) - set(pj["stages"][k - 1]["local"]))
                for k in range(1, pj["staging"]["s"]))
        T = sum(len(set(pj["stages"][k]["global"]) - set(pj["stages"][k - 1]["global"]))
                for k in range(1, pj["staging"]["s"]))
        assert pj["staging"]["cost"] == pytest.approx(S + cf * T)
    assert all(p == plans[0] for p in plans)


def _kcost(c, **opt):
    with A.Simulator(c.n, 0, 1, 0, **opt) as s:
        s.load_circuit(c.gates)
        s.plan()
        return s.plan_stats()["kernel_cost"]


@pytest.mark.parametrize("fam", ["qft", "ising", "qsvm", "wstate", "random"])
def test_kernelize_dp_unpruned_not_worse_than_ordered(fam):
    """Thm. dp-optimal: without pruning (T beyond any position's
    state count) the Kernelize DP alone is never worse than
    OrderedKernelize; the default Kernelize (cheapest valid of DP, Ordered and
    the front packing, R29) is never worse than either (E7's invariants)."""
    n = 12
    c = C.random_circuit(n, 40, 21, max_arity=2) if fam == "random" else C.make(fam, n)
    dp = _kcost(c, kernelizer=4, prune_T=0, ls_qubits=4)
    ordered = _kcost(c, kernelizer=1, ls_qubits=4)
    front = _kcost(c, kernelizer=3, ls_qubits=4)
    default = _kcost(c, kernelizer=0, ls_qubits=4)
    assert dp <= ordered
    assert default <= min(ordered, front)
