"""Pins of the planner oracles (oracle/planner.py, oracle/remap.py) against the
paper's definitions, theorems and worked examples."""
import itertools
import json
import os

import numpy as np
import pytest

from oracle import gates as OG, planner as P, remap as RM
from workloads import circuits as C

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# -------------------------------------------------------------- insularity
def test_insularity_definition_examples():
    """Def. Insular Qubit as quoted by SPEC S:L84-87."""
    assert OG.insular_qubits("Z") == {0}
    assert OG.insular_qubits("X") == {0}           # anti-diagonal
    assert OG.insular_qubits("H") == set()
    assert OG.insular_qubits("CX") == {0}          # control only
    assert OG.insular_qubits("CZ") == {0, 1}       # footnote: any qubit may control
    assert OG.insular_qubits("CP", (0.3,)) == {0, 1}
    assert OG.insular_qubits("CCX") == {0, 1}
    assert OG.insular_qubits("SWAP") == set()
    assert OG.insular_qubits("CU", (0.3, 0.2, 0.1, 0.05)) == {0}
    assert OG.insular_qubits("U3", (0.0, 0.2, 0.1)) == {0}   # diagonal U3
    assert OG.insular_qubits("RX", (np.pi,)) == {0}          # anti-diagonal
    assert OG.insular_kind("RX", (np.pi,)) == ("anti",)


# ------------------------------------------------------------ dependencies
def test_dependencies_examples():
    """ghz(3) -> {(0,1),(1,2)}; disjoint -> {}; qft(3) -> 6."""
    f = P.gate_facts(C.ghz(3))
    assert P.dependencies(f) == [(0, 1), (1, 2)]
    f = P.gate_facts(C.Circuit(2, [C.Gate("H", (0,)), C.Gate("H", (1,))]))
    assert P.dependencies(f) == []
    assert len(P.dependencies(P.gate_facts(C.qft(3)))) == 6


# ----------------------------------------------------------------- staging
def test_stage_single_stage_cost_zero():
    c = C.Circuit(4, [C.Gate("H", (0,)), C.Gate("CX", (0, 1))])
    plan = P.stage_bruteforce(c, L=2, Gq=2)
    assert plan.s == 1 and plan.cost == 0


def test_stage_ghz3_infeasible_at_one_stage():
    """SURVEY Q16 (correcting SPEC S:L182): ghz(3), L=2, G=1 is infeasible at
    s=1; optimum s=2, J = 1 + c, three-way tie; canonical pick ({q1},{q0})."""
    c = C.ghz(3)
    plan = P.stage_bruteforce(c, L=2, Gq=1, s_max=3, c=3)
    assert plan.s == 2 and plan.cost == 4
    assert plan.n_optimal == 3
    assert [sorted(g) for g in plan.globals] == [[1], [0]]
    assert plan.gate_stage == [0, 1, 1]  # H in stage 0 (q1 global); both CX in stage 1


def test_stage_six_h_gates():
    """6 H gates on 6 qubits, L=3, G=3, c=3 -> 2 stages,
    cost 3 * (1 + 3) = 12."""
    c = C.Circuit(6, [C.Gate("H", (q,)) for q in range(6)])
    plan = P.stage_bruteforce(c, L=3, Gq=3, s_max=2, c=3)
    assert plan.s == 2 and plan.cost == 12


def test_stage_qft6_unique_optimum():
    """qft(6) with L=3, G=3 -> s=2 with 3 swaps, unique."""
    plan = P.stage_bruteforce(C.qft(6), L=3, Gq=3, s_max=2, c=3)
    assert plan.s == 2 and plan.cost == 12 and plan.n_optimal == 1


@pytest.mark.parametrize("seed", range(12))
def test_maximal_execution_reaches_ilp_optimum(seed):
    """Lemma: for fixed per-stage sets the objective does not
    depend on F and the maximal F is feasible whenever any F is.  So the
    maximal-execution enumeration must equal the literal ILP enumeration in
    minimum s, minimum objective, and the set of optimal (A, B) sequences."""
    rng = np.random.default_rng(seed)
    n = 4 if seed % 2 else 3
    m = 4 if n == 3 else 3
    c = C.random_circuit(n, m, 100 + seed, kinds=("H", "X", "Z", "CX", "CZ", "RY"),
                         max_arity=2)
    L, Gq = n - 1, 1
    for s in (1, 2):
        obj, opt = P.ilp_enumerate(c, L, Gq, s, c=3)
        bf = P.stage_bruteforce(c, L, Gq, s_max=s, c=3)
        if obj is None:
            assert bf is None or bf.s > s
            continue
        assert bf is not None and bf.s <= s
        if bf.s == s:
            assert bf.cost == obj
            # the canonical plan is among the ILP optima
            assert (tuple(zip(bf.locals, bf.globals))) in [tuple(x) for x in opt]
        break


@pytest.mark.parametrize("seed", range(6))
def test_stage_monotone_in_L(seed):
    """more local qubits never need more stages."""
    c = C.random_circuit(6, 10, 300 + seed, kinds=("H", "CX", "CZ", "RZ", "U3"),
                         max_arity=2)
    prev = None
    for L in (3, 4, 5):
        plan = P.stage_bruteforce(c, L=L, Gq=6 - L, s_max=4, c=3)
        assert plan is not None
        if prev is not None:
            assert plan.s <= prev
        prev = plan.s


def test_stage_invariants_random():
    for seed in range(5):
        c = C.random_circuit(6, 12, 500 + seed, kinds=("H", "CX", "CZ", "CP", "T"),
                             max_arity=2)
        facts = P.gate_facts(c)
        plan = P.stage_bruteforce(c, L=4, Gq=2, s_max=4, c=3)
        for g, (qs, non) in enumerate(facts):
            k = plan.gate_stage[g]
            assert non <= plan.locals[k]
        for a, b in P.dependencies(facts):
            assert plan.gate_stage[a] <= plan.gate_stage[b]
        assert all(len(x) == 4 for x in plan.locals)
        assert P.stage_cost(plan.locals, plan.globals, 3) == plan.cost


def test_staging_cost_examples():
    """SPEC S:L199-202."""
    f = frozenset
    assert P.stage_cost([f({0, 1})], [f({2})], 3) == 0
    assert P.stage_cost([f({0, 1}), f({0, 1})], [f({2}), f({2})], 3) == 0
    assert P.stage_cost([f({0, 1, 2}), f({3, 4, 2})], [f({5}), f({0})], 3) == 5


# ---------------------------------------------------------- kernelization
def synthetic_model():
    """SPEC S:L350's synthetic model in integer units (x100): fusion_cost[q] =
    2^max(0, q-5), alpha = 0.8, gate_cost 0.05 / 0.08 / 0.12 by arity,
    q_max_fusion 7, q_max_shared 10, ls_qubits 3."""
    ar = {k: C.ARITY[k] for k in C.KINDS}
    return P.CostModel([100 * 2 ** max(0, q - 5) for q in range(1, 8)], 80,
                       {k: {1: 5, 2: 8, 3: 12}[ar[k]] for k in C.KINDS}, 7, 10, 3)


MODEL = synthetic_model()


def kseq(c, L=None):
    out = []
    for g in c.gates:
        ins = OG.insular_kind(g.kind, g.params)
        out.append(P.KGate(frozenset(g.qubits),
                           frozenset(q for q, t in zip(g.qubits, ins) if t is None),
                           g.kind))
    return out


def test_kernel_cost_examples():
    """SPEC S:L274-276 (in our integer units: synthetic model = SPEC x 100)."""
    ls = frozenset()
    seq = kseq(C.Circuit(3, [C.Gate("CX", (0, 1))]))
    cst, kind = P.kernel_cost(seq, MODEL, ls, L=30)
    assert (cst, kind) == (min(MODEL.fusion_cost[1],
                               MODEL.alpha + MODEL.gate_cost["CX"]),
                           "fusion" if MODEL.fusion_cost[1] <= MODEL.alpha + MODEL.gate_cost["CX"] else "shm")


def test_ordered_single_gate_and_disjoint_pair():
    seq = kseq(C.Circuit(12, [C.Gate("H", (0,))]))
    cost, segs = P.ordered_bruteforce(seq, MODEL, frozenset(), 12)
    assert len(segs) == 1 and cost == P.kernel_cost(seq, MODEL, frozenset(), 12)[0]
    # a model where doubling the qubits costs more than two kernels
    m2 = P.CostModel([100, 100, 1000, 1000], 10 ** 6, {k: 1 for k in C.KINDS}, 4, 4, 0)
    seq = kseq(C.Circuit(4, [C.Gate("CX", (0, 1)), C.Gate("CX", (2, 3))]))
    cost, segs = P.ordered_bruteforce(seq, m2, frozenset(), 4)
    assert cost == 200 and len(segs) == 2


def test_contiguous_segments_satisfy_constraint1():
    """Thm. contiguous, exhaustively on random sequences."""
    for seed in range(6):
        c = C.random_circuit(5, 9, 700 + seed, max_arity=3)
        qsets = [frozenset(g.qubits) for g in c.gates]
        for a in range(len(qsets)):
            for b in range(a + 1, len(qsets) + 1):
                assert P.satisfies_constraint1(set(range(a, b)), qsets)


def test_constraint1_paper_violations():
    """Fig. 'Kernel examples' prose.  Left: C[1], C[2], C[4]
    share q2 and only C[2] is excluded -> weak convexity fails.  Right: C[7]
    shares q1 with the kernel and is excluded, so the kernel's qubit set is
    fixed to {q0, q1}; adding C[9] on a new qubit breaks monotonicity."""
    q = frozenset
    left = [q({0}), q({1, 2}), q({2, 3}), q({4}), q({2, 5})]
    assert not P.satisfies_constraint1({1, 4}, left)
    assert P.satisfies_constraint1({1, 2, 4}, left)
    right = [q({5})] * 6 + [q({0, 1})] + [q({1, 3})] + [q({3})] + [q({1, 2})]
    # kernel {C6 (q0,q1), C9 (q1,q2)} after excluding C7 which shares q1
    assert not P.satisfies_constraint1({6, 9}, right)
    # without C9's new qubit it is fine: {C6} alone
    assert P.satisfies_constraint1({6}, right)


def test_extensible_definition_basics():
    q = frozenset
    qs = [q({0, 1}), q({1, 2}), q({3})]
    assert P.extensible_qubits(set(), 3, qs, 4) == q(range(4))      # empty kernel
    assert P.extensible_qubits({1, 2}, 3, qs, 4) == q(range(4))     # contiguous suffix
    # kernel {C0} after C1 (shares q1) is excluded: monotonicity fixes {q0,q1},
    # weak convexity removes q1
    assert P.extensible_qubits({0}, 2, qs, 4) == q({0})


@pytest.mark.parametrize("seed", range(8))
def test_ordered_bruteforce_plans_verify_and_bound(seed):
    """OrderedKernelize optimum verifies (Thm. contiguous) and is >= BF_opt
    over Constraint-1 kernel sets (Thm. dp-optimal's ordering of optima)."""
    c = C.random_circuit(6, 6, 900 + seed, max_arity=2)
    seq = kseq(c)
    m2 = P.CostModel([100, 120, 300, 700, 1500], 250,
                     {k: 10 for k in C.KINDS}, 5, 5, 0)
    cost, segs = P.ordered_bruteforce(seq, m2, frozenset(), 6)
    errs, recomputed = P.verify_plan([list(range(a, b)) for a, b, _ in segs],
                                     [k for _, _, k in segs], seq, m2, frozenset(), 6)
    assert errs == [] and recomputed == cost
    bf, part = P.kernel_bruteforce(seq, m2, frozenset(), 6)
    assert bf <= cost


# ------------------------------------------------------------------- remap
def test_remap_figure_counts():
    """Fig. qubit_remapping, L=R=G=1."""
    ident = [0, 1, 2]
    inter, intra = RM.comm_counts(3, 1, 1, ident, [1, 0, 2])  # local<->regional
    assert inter == 0 and intra == 4
    inter, intra = RM.comm_counts(3, 1, 1, ident, [2, 1, 0])  # local<->global
    assert inter == 4


def test_remap_is_a_permutation():
    rng = np.random.default_rng(3)
    n = 6
    psi = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    for _ in range(10):
        s1 = list(rng.permutation(n))
        s2 = list(rng.permutation(n))
        f1 = int(rng.integers(1 << n))
        f2 = int(rng.integers(1 << n))
        ph = RM.to_physical(psi, s1, f1)
        assert sorted(ph.tolist(), key=lambda z: (z.real, z.imag)) == \
            sorted(psi.tolist(), key=lambda z: (z.real, z.imag))
        back = RM.remap(RM.remap(ph, s1, f1, s2, f2), s2, f2, s1, f1)
        assert np.array_equal(back, ph)
        assert np.array_equal(RM.to_logical(RM.remap(ph, s1, f1, s2, f2), s2, f2), psi)
