"""Pins for the oracle's round-1 loose ends (VERDICT weak #1, "Next round"
item 2): every oracle function gets a check that a plausible mistake in it
would fail, independent of the function itself.

* Gate tables (both of the oracle's independent copies: the C table of
  sv_oracle.c via ``sim.gate_matrix`` and the NumPy table of ``gates.py``)
  against identities that fix their conventions from outside either table:
  rotations as matrix exponentials of Pauli matrices typed here
  (R_P(t) = exp(-i t P / 2)), U3 = e^{i(phi+lam)/2} RZ(phi) RY(theta) RZ(lam)
  (pins the phi/lambda order), U3(theta,-pi/2,pi/2) = RX(theta),
  U3(theta,0,0) = RY(theta), U3(0,0,lam) = P(lam), S^2 = Z, T^2 = S,
  HXH = Z, Y = iXZ, CU(theta,phi,lam,0) = controlled-U3,
  CU(0,0,0,gamma) = P(gamma) on the control, CX = (I x H) CZ (I x H),
  SWAP = CX CX' CX, CCX as a controlled-controlled X.
* ``verify_plan`` / ``orderable`` / ``conflicts``: negative cases that must
  be rejected (an X moved past the CX it controls -- P:L2459-2468 allows
  that only with a control-state flip, which the plan format does not
  carry; two non-diagonal gates on one qubit swapped; a CX target moved
  across a CZ on that qubit; non-partitions; size limits; Constraint 1),
  and a semantic soundness check: every gate order verify_plan accepts
  yields the same state as the circuit order under the oracle simulator.
* ``kernel_bruteforce`` (BF_opt, Thm. dp-optimal) on hand-solved
  instances where the optimum is non-contiguous (App. P:L2390-2393: the
  kind of kernel sequence OrderedKernelize cannot find) and where a
  Constraint-1-violating partition would be cheaper than the true optimum.
"""
import itertools
import math

import numpy as np
import pytest
from scipy.linalg import expm

from oracle import gates as OG
from oracle import planner as P
from oracle import sim as O
from workloads import circuits as C

# Pauli matrices and H typed here (not taken from either oracle table)
PX = np.array([[0, 1], [1, 0]], dtype=complex)
PY = np.array([[0, -1j], [1j, 0]], dtype=complex)
PZ = np.array([[1, 0], [0, -1]], dtype=complex)
I2 = np.eye(2, dtype=complex)
HH = np.array([[1, 1], [1, -1]], dtype=complex) / math.sqrt(2)

TABLES = {"c": O.gate_matrix, "numpy": OG.matrix}
ANGLES = [0.0, 0.37, 1.1, -2.3, math.pi, 5.9]


def close(a, b, tol=1e-13):
    return np.abs(np.asarray(a) - np.asarray(b)).max() <= tol


def kron_lsb(a, b):
    """Operator a on index bit 0 and b on index bit 1 (operand 0 = matrix
    LSB): index = b0 + 2 b1, so the Kronecker order is b x a."""
    return np.kron(b, a)


def controlled(v):
    """Control on index bit 0, target on index bit 1."""
    u = np.zeros((4, 4), dtype=complex)
    for c in range(2):
        for to in range(2):
            for ti in range(2):
                u[c + 2 * to, c + 2 * ti] = (v[to, ti] if c else (1.0 if to == ti else 0.0))
    return u


@pytest.mark.parametrize("tab", TABLES)
def test_fixed_gates(tab):
    M = TABLES[tab]
    assert close(M("X"), PX) and close(M("Y"), PY) and close(M("Z"), PZ)
    assert close(M("H"), HH)
    assert close(M("S") @ M("S"), M("Z"))
    assert close(M("T") @ M("T"), M("S"))
    assert close(M("S") @ M("SDG"), I2) and close(M("T") @ M("TDG"), I2)
    assert close(M("H") @ M("X") @ M("H"), M("Z"))
    assert close(M("H") @ M("Z") @ M("H"), M("X"))
    assert close(M("Y"), 1j * M("X") @ M("Z"))
    # Y|0> = i|1>  (sign of Y)
    assert close(M("Y") @ np.array([1, 0]), np.array([0, 1j]))


@pytest.mark.parametrize("tab", TABLES)
@pytest.mark.parametrize("t", ANGLES)
def test_rotations_are_pauli_exponentials(tab, t):
    M = TABLES[tab]
    assert close(M("RX", (t,)), expm(-1j * t / 2 * PX))
    assert close(M("RY", (t,)), expm(-1j * t / 2 * PY))
    assert close(M("RZ", (t,)), expm(-1j * t / 2 * PZ))
    # P(t) = diag(1, e^{it}) = e^{it/2} RZ(t)
    assert close(M("P", (t,)), np.exp(1j * t / 2) * expm(-1j * t / 2 * PZ))
    assert close(M("RY", (t,)), M("S") @ M("RX", (t,)) @ M("SDG"))


@pytest.mark.parametrize("tab", TABLES)
@pytest.mark.parametrize("th,ph,la", [(0.3, 1.2, -0.7), (2.2, -1.9, 0.4), (math.pi, 0.5, 2.5),
                                      (1.0, 0.0, 1.3)])
def test_u3_conventions(tab, th, ph, la):
    M = TABLES[tab]
    rz = lambda a: expm(-1j * a / 2 * PZ)  # noqa: E731
    ry = lambda a: expm(-1j * a / 2 * PY)  # noqa: E731
    # OpenQASM 2: U(theta, phi, lambda) = e^{i(phi+lambda)/2} RZ(phi) RY(theta) RZ(lambda)
    assert close(M("U3", (th, ph, la)), np.exp(1j * (ph + la) / 2) * rz(ph) @ ry(th) @ rz(la))
    assert close(M("U3", (th, -math.pi / 2, math.pi / 2)), M("RX", (th,)))
    assert close(M("U3", (th, 0.0, 0.0)), M("RY", (th,)))
    assert close(M("U3", (0.0, 0.0, la)), M("P", (la,)))
    # a phi <-> lambda swap would fail here (theta != 0, phi != lambda)
    if ph != la:
        assert not close(M("U3", (th, ph, la)), M("U3", (th, la, ph)), 1e-6)


@pytest.mark.parametrize("tab", TABLES)
def test_two_and_three_qubit_gates(tab):
    M = TABLES[tab]
    X, Z = PX, PZ
    assert close(M("CX"), controlled(X))
    assert close(M("CZ"), controlled(Z))
    for t in ANGLES:
        assert close(M("CP", (t,)), controlled(np.diag([1, np.exp(1j * t)])))
    # CX = (I x H_target) CZ (I x H_target)
    Ht = kron_lsb(I2, HH)
    assert close(M("CX"), Ht @ M("CZ") @ Ht)
    # SWAP = CX(0->1) CX(1->0) CX(0->1); CX(1->0) = SWAP-conjugate of CX
    sw = np.zeros((4, 4), dtype=complex)
    for b0 in range(2):
        for b1 in range(2):
            sw[b1 + 2 * b0, b0 + 2 * b1] = 1
    cx10 = sw @ controlled(X) @ sw
    assert close(M("SWAP"), controlled(X) @ cx10 @ controlled(X))
    assert close(M("SWAP"), sw)
    for th, ph, la in [(0.3, 1.2, -0.7), (2.2, -1.9, 0.4)]:
        assert close(M("CU", (th, ph, la, 0.0)), controlled(M("U3", (th, ph, la))))
        g = 0.9
        assert close(M("CU", (th, ph, la, g)), controlled(np.exp(1j * g) * M("U3", (th, ph, la))))
    for g in ANGLES:
        # CU(0,0,0,gamma) = P(gamma) on the control, identity on the target
        assert close(M("CU", (0.0, 0.0, 0.0, g)), kron_lsb(np.diag([1, np.exp(1j * g)]), I2))
    # CCX: controls index bits 0 and 1, target bit 2
    ccx = np.eye(8, dtype=complex)
    for b2 in range(2):
        i = 3 + 4 * b2
        j = 3 + 4 * (1 - b2)
        ccx[i, i] = 0
        ccx[i, j] = 1
    assert close(M("CCX"), ccx)


def test_oracle_simulator_uses_gate_on_right_qubits():
    """A gate on qubit q acts on bit q of the index with operand 0 as the
    matrix LSB: CX(2 -> 0) on |x> flips bit 0 iff bit 2 is set."""
    n = 3
    for x in range(8):
        psi = np.zeros(8, dtype=complex)
        psi[x] = 1
        out = O.simulate(C.Circuit(n, [C.Gate("CX", (2, 0))]), init=psi)
        y = x ^ 1 if (x >> 2) & 1 else x
        assert out[y] == 1 and np.count_nonzero(out) == 1


# ------------------------------------------------------------ plan checking
def kseq(gates, n):
    """Kernelizer input (reading R16: only diagonal-type operands insular)."""
    out = []
    for g in gates:
        ins = OG.insular_kind(g.kind, g.params)
        out.append(P.KGate(frozenset(g.qubits),
                           frozenset(q for q, t in zip(g.qubits, ins) if t != "diag"), g.kind))
    return out


def model(fus=(10, 10, 100, 1000), alpha=10 ** 6, qms=4, gate=1):
    return P.CostModel(list(fus), alpha, {k: gate for k in C.KINDS}, len(fus), qms, 0)


G_ = C.Gate


@pytest.mark.parametrize("lift", [False, True])
def test_verify_rejects_x_moved_past_its_control(lift):
    """X(q0) then CX(q0 -> q1): moving the X after the CX changes the result
    unless the CX's control state is flipped; a plan order
    that does so must be rejected."""
    gates = [G_("X", (0,)), G_("CX", (0, 1))]
    seq = kseq(gates, 2)
    m = model()
    assert P.verify_plan([[0], [1]], ["fusion"] * 2, seq, m, frozenset(), 2, lift=lift)[0] == []
    errs, _ = P.verify_plan([[1], [0]], ["fusion"] * 2, seq, m, frozenset(), 2, lift=lift)
    assert any("dependency" in e for e in errs)
    # and the two orders really differ
    a = O.simulate(C.Circuit(2, gates))
    b = O.simulate(C.Circuit(2, gates[::-1]))
    assert not np.allclose(a, b)


@pytest.mark.parametrize("lift", [False, True])
def test_verify_rejects_swapped_dense_gates_and_cx_target_vs_cz(lift):
    m = model()
    # two non-diagonal gates on one qubit
    seq = kseq([G_("H", (0,)), G_("U3", (0,), (0.3, 0.2, 0.1))], 1)
    errs, _ = P.verify_plan([[1], [0]], ["fusion"] * 2, seq, m, frozenset(), 1, lift=lift)
    assert errs
    # CX target q1 reordered across CZ(q1, q2): the target is non-insular
    seq = kseq([G_("CX", (0, 1)), G_("CZ", (1, 2))], 3)
    errs, _ = P.verify_plan([[1], [0]], ["fusion"] * 2, seq, m, frozenset(), 3, lift=lift)
    assert errs


def test_verify_lifting_allows_only_commuting_reorders():
    """CX(0 -> 1) and CZ(0, 2) share only q0, diagonal-type in both: with the
    insular lifting their order may change; without it (plain
    dependencies) it may not."""
    m = model()
    gates = [G_("CX", (0, 1)), G_("CZ", (0, 2))]
    seq = kseq(gates, 3)
    assert P.verify_plan([[1], [0]], ["fusion"] * 2, seq, m, frozenset(), 3, lift=True)[0] == []
    assert P.verify_plan([[1], [0]], ["fusion"] * 2, seq, m, frozenset(), 3, lift=False)[0] != []
    assert np.allclose(O.simulate(C.Circuit(3, gates)), O.simulate(C.Circuit(3, gates[::-1])))


def test_verify_rejects_malformed_plans():
    m = model(fus=(10, 10, 100), qms=2)
    seq = kseq([G_("H", (0,)), G_("CX", (0, 1)), G_("CCX", (0, 1, 2))], 3)
    # not a partition: gate 1 twice / gate 2 missing
    assert P.verify_plan([[0, 1], [1, 2]], ["fusion"] * 2, seq, m, frozenset(), 3)[0]
    assert P.verify_plan([[0, 1]], ["fusion"], seq, m, frozenset(), 3)[0]
    # fusion kernel over q_max_fusion = 3 qubits is fine, shm over q_max_shared = 2 is not
    assert P.verify_plan([[0, 1, 2]], ["fusion"], seq, m, frozenset(), 3)[0] == []
    errs, _ = P.verify_plan([[0, 1, 2]], ["shm"], seq, m, frozenset(), 3)
    assert any("active" in e for e in errs)
    m2 = model(fus=(10, 10), qms=4)
    errs, _ = P.verify_plan([[0, 1, 2]], ["fusion"], seq, m2, frozenset(), 3)
    assert any("fusion kernel" in e for e in errs)


def test_verify_rejects_constraint1_violation():
    """Fig. 'Kernel examples' left: C1, C2, C4 share q2 and C2 is
    excluded from the kernel {C1, C4} -> weak convexity fails."""
    gates = [G_("H", (0,)), G_("CX", (1, 2)), G_("CX", (2, 3)), G_("H", (4,)), G_("CX", (2, 5))]
    seq = kseq(gates, 6)
    m = model(fus=(10, 10, 100, 1000, 1000, 1000))
    kern = [[0], [1, 4], [2], [3]]
    errs, _ = P.verify_plan(kern, ["fusion"] * 4, seq, m, frozenset(), 6)
    assert any("Constraint 1" in e for e in errs)


def test_orderable_detects_cycles_and_returns_valid_orders():
    # H(q0) H(q0) H(q0): kernel {0, 2} and kernel {1} form a cycle
    seq = kseq([G_("H", (0,)), G_("H", (0,)), G_("H", (0,))], 1)
    assert P.orderable([[0, 2], [1]], seq) is None
    seq = kseq([G_("CX", (0, 1)), G_("CX", (2, 3)), G_("CX", (0, 1)), G_("CX", (2, 3))], 4)
    order = P.orderable([[1, 3], [0, 2]], seq)
    assert order is not None
    kern = [[[1, 3], [0, 2]][i] for i in order]
    assert P.verify_plan(kern, ["fusion"] * 2, seq, model(), frozenset(), 4)[0] == []


@pytest.mark.parametrize("seed", range(6))
def test_verify_accepted_orders_are_equivalent(seed):
    """Soundness of verify_plan's order check (Thm. dp-correct's notion,
    P:L1743): EVERY permutation of a small circuit that verify_plan accepts
    (each gate its own kernel, with and without lifting) gives the same state
    as the circuit order on a random input under the oracle simulator."""
    n = 3
    c = C.random_circuit(n, 6, 4200 + seed,
                         kinds=("H", "X", "Y", "Z", "S", "T", "RZ", "P", "CX", "CZ", "CP", "U3", "SWAP"),
                         max_arity=2)
    seq = kseq(c.gates, n)
    m = model()
    rng = np.random.default_rng(seed)
    psi0 = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    want = O.simulate(c, init=psi0)
    accepted = 0
    for perm in itertools.permutations(range(len(c.gates))):
        for lift in (False, True):
            errs, _ = P.verify_plan([[g] for g in perm], ["fusion"] * len(perm), seq, m,
                                    frozenset(), n, lift=lift)
            if errs:
                continue
            accepted += 1
            got = O.simulate(c, init=psi0, gates=[c.gates[g] for g in perm])
            assert np.abs(got - want).max() <= 1e-12, (perm, lift)
    assert accepted >= 2  # the identity order, with and without lifting


# ------------------------------------------------------------------- BF_opt
def test_kernel_bruteforce_noncontiguous_optimum():
    """Hand-solved: CX(0,1) CX(2,3) CX(0,1) CX(2,3) with fusion cost 10 for
    <= 2 qubits, 100 for 3, 1000 for 4 (shared-memory kernels priced out).
    Contiguous segmentations (OrderedKernelize) cannot merge the repeated
    pairs without taking 4 qubits: best 4 x 10 = 40.  The non-contiguous
    kernels {g0, g2}, {g1, g3} satisfy Constraint 1 (no qubit shared with the
    excluded gate in between; the excluded gate shares no qubit with the
    kernel) and cost 10 + 10 = 20, the unique optimum (P:L2390-2393's point:
    an ordering OrderedKernelize is not given)."""
    gates = [G_("CX", (0, 1)), G_("CX", (2, 3)), G_("CX", (0, 1)), G_("CX", (2, 3))]
    seq = kseq(gates, 4)
    m = model()
    bf, part = P.kernel_bruteforce(seq, m, frozenset(), 4)
    assert bf == 20
    assert sorted(sorted(k) for k in part) == [[0, 2], [1, 3]]
    oc, _ = P.ordered_bruteforce(seq, m, frozenset(), 4)
    assert oc == 40


def test_kernel_bruteforce_respects_constraint1():
    """Hand-solved: CX(0,1) CX(1,2) CX(0,1).  {g0, g2} would cost 10 + 10 for
    g1 = 20, but g0, g1, g2 share q1 with g1 excluded (weak convexity,
    P:L1685) -- and the kernels could not be ordered anyway.  Admissible:
    three singletons (30) or {g0, g1} / {g1, g2} with 3 qubits (100 + 10).
    BF_opt = 30."""
    gates = [G_("CX", (0, 1)), G_("CX", (1, 2)), G_("CX", (0, 1))]
    seq = kseq(gates, 3)
    bf, part = P.kernel_bruteforce(seq, model(), frozenset(), 3)
    assert bf == 30
    assert sorted(sorted(k) for k in part) == [[0], [1], [2]]


def test_kernel_bruteforce_shared_memory_kind():
    """Hand-solved, shared-memory kernels allowed: H on q0..q3 then CZ(0,3),
    fusion 10/20/400/800 by qubit count, alpha = 25, 1 per gate,
    q_max_shared = 4.  All five gates in one shared-memory kernel: 25 + 5 =
    30.  The best all-fusion plan is {H0, H3, CZ} (2 qubits: 20) + {H1, H2}
    (2 qubits: 20) = 40; one fusion kernel of all four qubits is 800; a
    shared-memory kernel of fewer gates plus fusion kernels pays alpha and
    at least 10 more.  BF_opt = 30, unique."""
    gates = [G_("H", (0,)), G_("H", (1,)), G_("H", (2,)), G_("H", (3,)), G_("CZ", (0, 3))]
    seq = kseq(gates, 4)
    m = P.CostModel([10, 20, 400, 800], 25, {k: 1 for k in C.KINDS}, 4, 4, 0)
    bf, part = P.kernel_bruteforce(seq, m, frozenset(), 4)
    assert bf == 30
    assert part == [[0, 1, 2, 3, 4]]
    assert P.kernel_cost([seq[i] for i in range(5)], m, frozenset(), 4) == (30, "shm")
