"""O2: brute-force planner oracles (staging, kernel segmentation, Constraint 1).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Everything here is enumeration straight from the paper's definitions, for
tiny instances only (n <= 8, m <= ~14).

Staging (PAPER.md §"Circuit Staging")
---------------------------------------------------
``ilp_enumerate``     literal enumeration of the binary ILP (objective
                      P:L1491, constraints c1-c6 P:L1495-1502) over A, B, F
                      (S, T take their minimal feasible values).  Only for
                      n <= 4, m <= 4, s <= 2.  Pinned by the paper's objective
                      definition and SPEC's worked counts.
``stage_bruteforce``  enumeration of per-stage (local, global) qubit sets with
                      *maximal execution* (each gate finishes in the first
                      stage where c3/c4 allow it).  The lemma that this reaches
                      the ILP optimum is pinned against
                      ``ilp_enumerate`` in tests.  Minimum s (Thm. ilp-optimal,
                      P:L1539), then minimum objective (Eq. P:L1477), then the
                      canonical tie-break of DESIGN.md reading R5: the
                      lexicographically smallest tuple of per-stage global
                      bitmasks (then local bitmasks).

Kernelization (PAPER.md §"Circuit Kernelization", App. P:L2348)
-------------------------------------------------------------------------------
``ordered_bruteforce``  all 2^{m-1} contiguous segmentations (the optimum
                        OrderedKernelize reaches, P:L2362 / Problem 1
                        P:L1639-1653); canonical tie-break = lexicographically
                        smallest tuple of segment starts read from the last
                        segment backwards (reading R21), fusion preferred on a
                        kind tie.
``satisfies_constraint1``  Constraint 1 by its quantifiers.
``extensible_qubits``   Def. "Extensible qubit" by its
                        quantifiers.
``kernel_bruteforce``   BF_opt: all set partitions into kernels satisfying
                        Constraint 1 whose concatenation can be ordered
                        topologically (Thm. dp-correct's notion),
                        minimum total cost.  Only a bound for Kernelize
                        (Thm. dp-optimal): "parity unpinned" beyond
                        BF_opt <= Kernelize <= OrderedKernelize.
``verify_plan``         partition + Constraint 1 + topological equivalence +
                        size limits + cost recomputation.
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple

from . import gates as G

INF = float("inf")


# ----------------------------------------------------------------------------
# circuit facts by definition
# ----------------------------------------------------------------------------
def gate_facts(circuit):
    """Per gate: (qubits tuple, frozenset of non-insular qubits)."""
    out = []
    for g in circuit.gates:
        ins = G.insular_kind(g.kind, g.params)
        non = frozenset(q for q, t in zip(g.qubits, ins) if t is None)
        out.append((tuple(g.qubits), non))
    return out


def dependencies(facts) -> List[Tuple[int, int]]:
    """E: adjacent gate pairs on the same qubit, by an O(m^2) scan."""
    edges = set()
    m = len(facts)
    for b in range(m):
        for q in facts[b][0]:
            for a in range(b - 1, -1, -1):
                if q in facts[a][0]:
                    edges.add((a, b))
                    break
    return sorted(edges)


def _mask(s) -> int:
    v = 0
    for q in s:
        v |= 1 << q
    return v


# ----------------------------------------------------------------------------
# staging
# ----------------------------------------------------------------------------
def maximal_execution(facts, preds, done, local) -> List[bool]:
    """Finish every gate whose predecessors are finished (c4) and whose
    non-insular qubits are local in this stage (c3), to a fixpoint."""
    done = list(done)
    changed = True
    while changed:
        changed = False
        for g, (qs, non) in enumerate(facts):
            if done[g]:
                continue
            if all(done[p] for p in preds[g]) and non <= local:
                done[g] = True
                changed = True
    return done


def stage_cost(locals_, globals_, c) -> float:
    """Eq. P:L1477: sum_{i>=1} |Q_i^loc \\ Q_{i-1}^loc| + c |Q_i^glob \\ Q_{i-1}^glob|."""
    j = 0
    for i in range(1, len(locals_)):
        j += len(locals_[i] - locals_[i - 1]) + c * len(globals_[i] - globals_[i - 1])
    return j


@dataclass
class StagePlan:
    s: int
    cost: float
    locals: List[frozenset]
    globals: List[frozenset]
    gate_stage: List[int]
    n_optimal: int = 1


def stage_bruteforce(circuit, L: int, Gq: int, s_max: int = 3, c: float = 3,
                     facts=None) -> Optional[StagePlan]:
    n = circuit.n
    R = n - L - Gq
    assert R >= 0
    facts = facts if facts is not None else gate_facts(circuit)
    m = len(facts)
    preds = [[] for _ in range(m)]
    for a, b in dependencies(facts):
        preds[b].append(a)
    # every (local, global) choice for one stage
    choices = []
    for loc in itertools.combinations(range(n), L):
        rest = [q for q in range(n) if q not in loc]
        for glob in itertools.combinations(rest, Gq):
            choices.append((frozenset(loc), frozenset(glob)))
    for s in range(1, s_max + 1):
        best = None
        n_opt = 0
        for seq in itertools.product(choices, repeat=s):
            done = [False] * m
            stage_of = [-1] * m
            for k, (loc, _) in enumerate(seq):
                nd = maximal_execution(facts, preds, done, loc)
                for g in range(m):
                    if nd[g] and not done[g]:
                        stage_of[g] = k
                done = nd
            if not all(done):
                continue
            locs = [x[0] for x in seq]
            globs = [x[1] for x in seq]
            j = stage_cost(locs, globs, c)
            key = (j, tuple(_mask(x) for x in globs), tuple(_mask(x) for x in locs))
            if best is None or key < best[0]:
                if best is None or key[0] < best[0][0]:
                    n_opt = 1
                else:
                    n_opt += 1
                best = (key, StagePlan(s, j, locs, globs, stage_of))
            elif key[0] == best[0][0]:
                n_opt += 1
        if best is not None:
            best[1].n_optimal = n_opt
            return best[1]
    return None


def ilp_enumerate(circuit, L: int, Gq: int, s: int, c: float = 3, facts=None):
    """Literal enumeration of the ILP for tiny instances.

    Returns (min objective or None if infeasible, list of optimal (A, B)
    stage-set sequences).  S and T take their minimal values allowed by
    c1/cdeft (the objective is minimised, so any larger value is dominated)."""
    n = circuit.n
    facts = facts if facts is not None else gate_facts(circuit)
    m = len(facts)
    edges = dependencies(facts)
    sets = []
    for loc in itertools.combinations(range(n), L):
        rest = [q for q in range(n) if q not in loc]
        for glob in itertools.combinations(rest, Gq):
            sets.append((frozenset(loc), frozenset(glob)))  # c6, cag hold
    best = None
    opt = []
    for AB in itertools.product(sets, repeat=s):
        for bits in range(1 << (m * s)):
            F = [[(bits >> (g * s + k)) & 1 for k in range(s)] for g in range(m)]
            ok = True
            for g in range(m):
                if F[g][s - 1] != 1:          # c5
                    ok = False
                    break
                for k in range(s - 1):        # c2
                    if F[g][k] > F[g][k + 1]:
                        ok = False
                        break
                if not ok:
                    break
                for k in range(s):            # c3, F_{g,-1} = 0 (reading R3)
                    prev = F[g][k - 1] if k > 0 else 0
                    for q in facts[g][1]:
                        a = 1 if q in AB[k][0] else 0
                        if F[g][k] > prev + a:
                            ok = False
                            break
                    if not ok:
                        break
                if not ok:
                    break
            if ok:
                for (g1, g2) in edges:        # c4
                    for k in range(s):
                        if F[g1][k] < F[g2][k]:
                            ok = False
                            break
                    if not ok:
                        break
            if not ok:
                continue
            obj = 0
            for k in range(s - 1):
                for q in range(n):
                    S = max(0, (q in AB[k + 1][0]) - (q in AB[k][0]))
                    T = max(0, (q in AB[k + 1][1]) - (q in AB[k][1]))
                    obj += S + c * T
            if best is None or obj < best:
                best, opt = obj, [AB]
            elif obj == best and AB not in opt:
                opt.append(AB)
    return best, opt


def ilp_highs(circuit, L: int, Gq: int, s: int, c: float = 3, facts=None, time_limit=120.0):
    """The paper's staging ILP, literally (objective Eq. P:L1491, constraints
    c1, cdeft, c2, c3, c4, c5, cag, c6 at P:L1495-1502, F_{g,-1} = 0 per
    reading R3), with R = n - L - G regional qubits, handed to an
    off-the-shelf ILP solver as the paper does (it used PuLP +
    HiGHS; here HiGHS through scipy.optimize.milp).  For instances far beyond
    ``ilp_enumerate``.  Returns (objective or None if infeasible, optimal:
    bool, A as s x n 0/1 list of local sets)."""
    import numpy as np
    from scipy.optimize import Bounds, LinearConstraint, milp
    from scipy.sparse import lil_matrix
    n = circuit.n
    facts = facts if facts is not None else gate_facts(circuit)
    m = len(facts)
    edges = dependencies(facts)
    # variable layout: A[q,k], B[q,k], F[g,k], S[q,k<s-1], T[q,k<s-1]
    nA = n * s
    oA, oB, oF = 0, nA, 2 * nA
    oS = oF + m * s
    oT = oS + n * (s - 1)
    nv = oT + n * (s - 1)
    A_ = lambda q, k: oA + q * s + k  # noqa: E731
    B_ = lambda q, k: oB + q * s + k  # noqa: E731
    F_ = lambda g, k: oF + g * s + k  # noqa: E731
    S_ = lambda q, k: oS + q * (s - 1) + k  # noqa: E731
    T_ = lambda q, k: oT + q * (s - 1) + k  # noqa: E731
    cost = np.zeros(nv)
    for q in range(n):
        for k in range(s - 1):
            cost[S_(q, k)] = 1.0
            cost[T_(q, k)] = c
    rows = []  # (coeffs dict, lo, hi)
    for q in range(n):
        for k in range(s - 1):
            rows.append(({A_(q, k + 1): 1, A_(q, k): -1, S_(q, k): -1}, -np.inf, 0))   # c1
            rows.append(({B_(q, k + 1): 1, B_(q, k): -1, T_(q, k): -1}, -np.inf, 0))   # cdeft
    for g in range(m):
        for k in range(s - 1):
            rows.append(({F_(g, k): 1, F_(g, k + 1): -1}, -np.inf, 0))                  # c2
        for q in facts[g][1]:
            for k in range(s):
                d = {F_(g, k): 1, A_(q, k): -1}
                if k > 0:
                    d[F_(g, k - 1)] = -1                                                # c3
                rows.append((d, -np.inf, 0))
        rows.append(({F_(g, s - 1): 1}, 1, 1))                                          # c5
    for g1, g2 in edges:
        for k in range(s):
            rows.append(({F_(g1, k): 1, F_(g2, k): -1}, 0, np.inf))                     # c4
    for q in range(n):
        for k in range(s):
            rows.append(({A_(q, k): 1, B_(q, k): 1}, -np.inf, 1))                       # cag
    for k in range(s):
        rows.append(({A_(q, k): 1 for q in range(n)}, L, L))                            # c6
        rows.append(({B_(q, k): 1 for q in range(n)}, Gq, Gq))
    M = lil_matrix((len(rows), nv))
    lo = np.empty(len(rows))
    hi = np.empty(len(rows))
    for i, (d, a, b) in enumerate(rows):
        for j, v in d.items():
            M[i, j] = v
        lo[i], hi[i] = a, b
    res = milp(cost, constraints=LinearConstraint(M.tocsr(), lo, hi),
               integrality=np.ones(nv), bounds=Bounds(0, 1),
               options={"time_limit": time_limit, "disp": False})
    if res.status == 2:  # infeasible
        return None, True, None
    if res.x is None:
        return None, False, None
    x = np.round(res.x).astype(int)
    locs = [[q for q in range(n) if x[A_(q, k)]] for k in range(s)]
    return float(round(res.fun, 9)), res.status == 0, locs


# ----------------------------------------------------------------------------
# kernel cost model
# ----------------------------------------------------------------------------
@dataclass
class CostModel:
    fusion_cost: List[int]          # index q-1
    alpha: int
    gate_cost: Dict[str, int]
    q_max_fusion: int
    q_max_shared: int
    ls_qubits: int

    @staticmethod
    def from_json(d) -> "CostModel":
        return CostModel(list(d["fusion_cost"]), d["alpha"], dict(d["gate_cost"]),
                         d["q_max_fusion"], d["q_max_shared"], d["ls_qubits"])


@dataclass
class KGate:
    """One gate as the kernelizer sees it inside a stage."""
    qubits: frozenset       # its qubits that are local in the stage (Q13)
    active: frozenset       # its non-insular local qubits
    kind: str


def kernel_cost(kgates: Sequence[KGate], model: CostModel, ls_set: frozenset,
                L: int) -> Tuple[float, str]:
    """Cost of one kernel = min over the kinds that fit (fusion preferred on a
    tie).  Fusion: fusion_cost[|Qubits|].  Shared memory:
    alpha + sum Cost(g) when |active U LSB| <= q_max_shared."""
    qs = frozenset().union(*[g.qubits for g in kgates])
    act = frozenset().union(*[g.active for g in kgates]) | ls_set
    qmf = min(model.q_max_fusion, L)
    qms = min(model.q_max_shared, L)
    f = model.fusion_cost[len(qs) - 1] if 1 <= len(qs) <= qmf else INF
    s = model.alpha + sum(model.gate_cost[g.kind] for g in kgates) \
        if len(act) <= qms else INF
    if f <= s:
        return f, "fusion"
    return s, "shm"


def ordered_bruteforce(seq: Sequence[KGate], model: CostModel, ls_set, L):
    """Minimum over all contiguous segmentations; returns (cost, segments)
    where segments = [(start, end_exclusive, kind)]."""
    m = len(seq)
    best = None
    for cuts in range(1 << max(m - 1, 0)):
        starts = [0] + [i + 1 for i in range(m - 1) if (cuts >> i) & 1]
        ends = starts[1:] + [m]
        total = 0
        segs = []
        for a, b in zip(starts, ends):
            cst, kind = kernel_cost(seq[a:b], model, ls_set, L)
            total += cst
            segs.append((a, b, kind))
        if total == INF:
            continue
        key = (total, tuple(reversed(starts)))
        if best is None or key < best[0]:
            best = (key, segs)
    if best is None:
        return INF, None
    return best[0][0], best[1]


# ----------------------------------------------------------------------------
# Constraint 1 / extensible qubits / plan checking
# ----------------------------------------------------------------------------
def satisfies_constraint1(K: set, qsets: Sequence[frozenset]) -> bool:
    """Weak convexity and monotonicity of P:L1685-1699, by their quantifiers."""
    m = len(qsets)
    for j1 in range(m):
        if j1 not in K:
            continue
        for j2 in range(j1 + 1, m):
            if j2 in K:
                continue
            for j3 in range(j2 + 1, m):
                if j3 in K and (qsets[j1] & qsets[j2] & qsets[j3]):
                    return False
    allq = frozenset().union(*[qsets[j] for j in K]) if K else frozenset()
    for j in range(m):
        if j in K:
            continue
        before = [i for i in K if i < j]
        qb = frozenset().union(*[qsets[i] for i in before]) if before else frozenset()
        if qsets[j] & qb and allq != qb:
            return False
    return True


def extensible_qubits(K: set, i: int, qsets: Sequence[frozenset], n: int) -> frozenset:
    """Def. 5: the qubits q for which adding a gate on q to
    K|<i satisfies Constraint 1."""
    Ki = {j for j in K if j < i}
    out = set()
    for q in range(n):
        ok = True
        for j1 in Ki:
            for j2 in range(j1 + 1, i):
                if j2 not in Ki and q in qsets[j1] and q in qsets[j2]:
                    ok = False
        for j in range(i):
            if j in Ki:
                continue
            before = [x for x in Ki if x < j]
            qb = frozenset().union(*[qsets[x] for x in before]) if before else frozenset()
            if qsets[j] & qb and q not in qb:
                ok = False
        if ok:
            out.add(q)
    return frozenset(out)


def conflicts(a: KGate, b: KGate, lift: bool) -> bool:
    """Two gates must keep their relative order iff they share a qubit
    (plain), or -- with the insular lifting of P:L2454 -- iff they
    share a qubit that is non-insular to at least one of them."""
    shared = a.qubits & b.qubits
    if not lift:
        return bool(shared)
    return bool(shared & (a.active | b.active))


def orderable(kernels: Sequence[Sequence[int]], seq: Sequence[KGate], lift=False):
    """Is there an order of the kernels (each kept in original gate order)
    whose concatenation is topologically equivalent to seq?  Returns one such
    order (list of kernel indices) or None."""
    where = {}
    for ki, K in enumerate(kernels):
        for g in K:
            where[g] = ki
    nk = len(kernels)
    succ = [set() for _ in range(nk)]
    m = len(seq)
    for a in range(m):
        for b in range(a + 1, m):
            if conflicts(seq[a], seq[b], lift) and where[a] != where[b]:
                succ[where[a]].add(where[b])
    indeg = [0] * nk
    for a in range(nk):
        for b in succ[a]:
            indeg[b] += 1
    ready = [k for k in range(nk) if indeg[k] == 0]
    order = []
    while ready:
        ready.sort()
        k = ready.pop(0)
        order.append(k)
        for b in succ[k]:
            indeg[b] -= 1
            if indeg[b] == 0:
                ready.append(b)
    return order if len(order) == nk else None


def _set_partitions(items):
    if not items:
        yield []
        return
    first, rest = items[0], items[1:]
    for part in _set_partitions(rest):
        for i in range(len(part)):
            yield part[:i] + [[first] + part[i]] + part[i + 1:]
        yield [[first]] + part


def kernel_bruteforce(seq: Sequence[KGate], model: CostModel, ls_set, L):
    """BF_opt: minimum total cost over all kernel sets satisfying Constraint 1
    that admit a topologically equivalent order (plain dependencies)."""
    qsets = [g.qubits for g in seq]
    best = INF
    best_part = None
    for part in _set_partitions(list(range(len(seq)))):
        part = [sorted(k) for k in part]
        if not all(satisfies_constraint1(set(k), qsets) for k in part):
            continue
        total = 0
        for k in part:
            total += kernel_cost([seq[i] for i in k], model, ls_set, L)[0]
        if total >= best:
            continue
        if orderable(part, seq) is None:
            continue
        best, best_part = total, part
    return best, best_part


def verify_plan(kernels: Sequence[Sequence[int]], kinds: Sequence[str],
                seq: Sequence[KGate], model: CostModel, ls_set, L,
                lift: bool = False, check_constraint1: bool = True):
    """partition, Constraint 1, size limits, and that the
    concatenation in the GIVEN kernel order is topologically equivalent to seq.
    Returns a list of violation strings (empty = ok) and the recomputed cost."""
    errs = []
    m = len(seq)
    seen = sorted(g for K in kernels for g in K)
    if seen != list(range(m)):
        errs.append("not a partition of the stage's gates")
        return errs, INF
    qsets = [g.qubits for g in seq]
    total = 0
    qmf = min(model.q_max_fusion, L)
    qms = min(model.q_max_shared, L)
    for K, kind in zip(kernels, kinds):
        if check_constraint1 and not lift and not satisfies_constraint1(set(K), qsets):
            errs.append(f"kernel {list(K)} violates Constraint 1")
        qs = frozenset().union(*[seq[i].qubits for i in K])
        act = frozenset().union(*[seq[i].active for i in K]) | ls_set
        if kind == "fusion":
            if not 1 <= len(qs) <= qmf:
                errs.append(f"fusion kernel {list(K)} has {len(qs)} qubits")
            else:
                total += model.fusion_cost[len(qs) - 1]
        else:
            if len(act) > qms:
                errs.append(f"shm kernel {list(K)} has {len(act)} active qubits")
            total += model.alpha + sum(model.gate_cost[seq[i].kind] for i in K)
    pos = {}
    p = 0
    for K in kernels:
        for g in sorted(K):
            pos[g] = p
            p += 1
    for a in range(m):
        for b in range(a + 1, m):
            if conflicts(seq[a], seq[b], lift) and pos[a] > pos[b]:
                errs.append(f"order violates dependency {a}->{b}")
    return errs, total
