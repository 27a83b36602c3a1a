"""Pins of the simulation oracle O1 (oracle/sv_oracle.c) against things the
paper and mathematics fix -- never against itself."""
import cmath
import json
import math
import os

import numpy as np
import pytest

from oracle import einsum_sim, gates as OG, sim
from workloads import circuits as C

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_gate_counts_match_paper_table():
    """Generators reproduce Table 'benchmark circuits'."""
    d = json.load(open(os.path.join(GOLD, "benchmark_gate_counts.json")))
    for fam in C.FAMILIES:
        for n, want in zip(d["qubits"], d["counts"][fam]):
            assert C.expected_gate_count(fam, n) == want, (fam, n)
            if n <= 30:
                assert len(C.make(fam, n)) == want, (fam, n)


def test_eq2_index_pairs():
    """Eq. 2: a 1-qubit gate on q mixes exactly the pair
    (f(i), f(i)+2^q); checked on printed/hand-evaluated values."""
    d = json.load(open(os.path.join(GOLD, "eq2_index_examples.json")))
    rng = np.random.default_rng(7)
    for ex in d["examples"]:
        n, q, i = ex["n"], ex["q"], ex["i"]
        f = (2 ** (q + 1)) * (i // 2 ** q) + (i % 2 ** q)
        assert [f, f + 2 ** q] == ex["pair"]
        psi = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
        u3 = (0.7, 0.3, -1.1)
        out = sim.simulate(C.Circuit(n, [C.Gate("U3", (q,), u3)]), init=psi)
        U = OG.matrix("U3", u3)
        a, b = ex["pair"]
        np.testing.assert_allclose([out[a], out[b]], U @ np.array([psi[a], psi[b]]),
                                   atol=1e-14)
        # every other pair is untouched by this pair's update rule
        others = [x for x in range(1 << n) if x not in (a, b)]
        for x in others:
            partner = x ^ (1 << q)
            lo, hi = min(x, partner), max(x, partner)
            want = (U @ np.array([psi[lo], psi[hi]]))[0 if x == lo else 1]
            assert abs(out[x] - want) < 1e-14


@pytest.mark.parametrize("n", [1, 2, 5, 10, 16])
def test_ghz_closed_form(n):
    psi = sim.simulate(C.ghz(n))
    want = np.zeros(1 << n, dtype=complex)
    want[0] = want[-1] = 1 / math.sqrt(2)
    assert np.abs(psi - want).max() < 1e-14


@pytest.mark.parametrize("n", [2, 3, 4, 7, 12])
def test_wstate_closed_form(n):
    psi = sim.simulate(C.wstate(n))
    want = np.zeros(1 << n, dtype=complex)
    for j in range(n):
        want[1 << j] = 1 / math.sqrt(n)
    assert np.abs(psi - want).max() < 1e-13


@pytest.mark.parametrize("n", [3, 5, 9, 12])
def test_graphstate_closed_form(n):
    c = C.graphstate(n)
    edges = [g.qubits for g in c.gates if g.kind == "CZ"]
    assert len(edges) == n
    psi = sim.simulate(c)
    x = np.arange(1 << n)
    par = np.zeros(1 << n, dtype=np.int64)
    for a, b in edges:
        par += ((x >> a) & 1) * ((x >> b) & 1)
    want = (2.0 ** (-n / 2)) * (-1.0) ** par
    assert np.abs(psi - want).max() < 1e-13


def _rev(x, n):
    return int(format(x, f"0{n}b")[::-1], 2)


@pytest.mark.parametrize("n", [3, 5, 8])
def test_qft_basis_states_closed_form(n):
    """QFT without swaps maps |x> to 2^{-n/2} sum_y exp(+2 pi i rev_n(x) y / 2^n) |y>
    (DFT of the bit-reversed input)."""
    y = np.arange(1 << n)
    for x in range(1 << n):
        psi = sim.simulate(C.prepend_basis(C.qft(n), x))
        want = (2.0 ** (-n / 2)) * np.exp(2j * np.pi * _rev(x, n) * y / 2 ** n)
        assert np.abs(psi - want).max() < 1e-13, x


def test_qft_large_sampled():
    n = 18
    x = 0b101100111000110101
    psi = sim.simulate(C.prepend_basis(C.qft(n), x))
    y = np.arange(1 << n)
    want = (2.0 ** (-n / 2)) * np.exp(2j * np.pi * _rev(x, n) * y / 2 ** n)
    assert np.abs(psi - want).max() < 1e-12


def _kron_full(n, kind, params, qubits):
    """Independent construction of the 2^n x 2^n operator of one gate:
    U = sum_{a,b} U[a,b] |a><b| on the gate's qubits, expanded as a sum of
    Kronecker products of single-site operators (site n-1 leftmost)."""
    U = OG.matrix(kind, params)
    k = len(qubits)
    full = np.zeros((1 << n, 1 << n), dtype=complex)
    e = [np.array([[1, 0], [0, 0]]), np.array([[0, 1], [0, 0]]),
         np.array([[0, 0], [1, 0]]), np.array([[0, 0], [0, 1]])]
    for a in range(1 << k):
        for b in range(1 << k):
            if U[a, b] == 0:
                continue
            op = np.array([[1.0 + 0j]])
            for site in range(n - 1, -1, -1):
                if site in qubits:
                    j = qubits.index(site)
                    aj, bj = (a >> j) & 1, (b >> j) & 1
                    op = np.kron(op, e[2 * aj + bj])
                else:
                    op = np.kron(op, np.eye(2))
            full += U[a, b] * op
    return full


@pytest.mark.parametrize("seed", range(4))
def test_full_unitary_matches_kronecker_products(seed):
    n = 5
    c = C.random_circuit(n, 12, seed)
    M = np.eye(1 << n, dtype=complex)
    for g in c.gates:
        M = _kron_full(n, g.kind, g.params, list(g.qubits)) @ M
    assert np.abs(M @ M.conj().T - np.eye(1 << n)).max() < 1e-12
    for j in range(1 << n):
        ej = np.zeros(1 << n, dtype=complex)
        ej[j] = 1
        col = sim.simulate(c, init=ej)
        assert np.abs(col - M[:, j]).max() < 1e-13


def test_every_kind_matrix_is_unitary_and_tables_agree():
    for k in C.KINDS:
        p = OG._dummy_params(k)
        u = sim.gate_matrix(k, p)
        assert np.abs(u @ u.conj().T - np.eye(u.shape[0])).max() < 1e-12
        assert np.abs(u - OG.matrix(k, p)).max() < 1e-15


@pytest.mark.parametrize("fam", C.FAMILIES)
def test_mirror_returns_to_zero(fam):
    c = C.mirror(C.make(fam, 10))
    psi = sim.simulate(c)
    assert abs(abs(psi[0]) ** 2 - 1) < 1e-12
    assert np.abs(psi[1:]).max() < 1e-12


@pytest.mark.parametrize("seed", range(3))
def test_mirror_random(seed):
    c = C.mirror(C.random_circuit(7, 40, seed))
    psi = sim.simulate(c)
    assert abs(psi[0] - 1) < 1e-12


@pytest.mark.parametrize("fam", C.FAMILIES)
def test_o1_equals_einsum_o1prime(fam):
    c = C.make(fam, 11)
    a = sim.simulate(c)
    b = einsum_sim.simulate(c)
    assert np.abs(a - b).max() < 1e-13
    assert abs(sim.norm2(a, c.n) - 1) < 1e-12 * len(c)


@pytest.mark.parametrize("seed", range(4))
def test_o1_equals_einsum_random(seed):
    c = C.random_circuit(9, 60, seed)
    rng = np.random.default_rng(seed)
    psi0 = rng.normal(size=512) + 1j * rng.normal(size=512)
    psi0 /= np.linalg.norm(psi0)
    a = sim.simulate(c, init=psi0)
    b = einsum_sim.simulate(c, init=psi0)
    assert np.abs(a - b).max() < 1e-13


def test_textbook_single_gate_examples():
    """H|0> = (|0>+|1>)/sqrt2; CX(control q0, target q1) on
    |q1=0,q0=1> gives |11>."""
    psi = sim.simulate(C.Circuit(1, [C.Gate("H", (0,))]))
    assert np.allclose(psi, [1 / math.sqrt(2)] * 2, atol=1e-15)
    psi = sim.simulate(C.Circuit(2, [C.Gate("X", (0,)), C.Gate("CX", (0, 1))]))
    assert abs(psi[3] - 1) < 1e-15
    # control = 0 leaves the target alone
    psi = sim.simulate(C.Circuit(2, [C.Gate("X", (1,)), C.Gate("CX", (0, 1))]))
    assert abs(psi[2] - 1) < 1e-15
    # CCX fires only when both controls are 1
    psi = sim.simulate(C.Circuit(3, [C.Gate("X", (0,)), C.Gate("X", (1,)),
                                     C.Gate("CCX", (0, 1, 2))]))
    assert abs(psi[7] - 1) < 1e-15
    # SWAP exchanges the qubits
    psi = sim.simulate(C.Circuit(3, [C.Gate("X", (0,)), C.Gate("SWAP", (0, 2))]))
    assert abs(psi[4] - 1) < 1e-15
    # RZ vs P differ by a global phase only
    a = sim.simulate(C.Circuit(1, [C.Gate("H", (0,)), C.Gate("RZ", (0,), (0.4,))]))
    b = sim.simulate(C.Circuit(1, [C.Gate("H", (0,)), C.Gate("P", (0,), (0.4,))]))
    assert np.allclose(a * cmath.exp(0.2j), b, atol=1e-15)
