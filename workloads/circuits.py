"""Seeded synthetic circuit generators shaped like the paper's benchmark suite.

This module is INPUT GENERATION ONLY.  It is shared by the CUDA product path
(bench.py, the Python binding tests) and by the CPU oracle (oracle/), and
therefore holds none of the method's arithmetic: no gate matrices, no
insularity rules, no staging, no kernelization.  A circuit is a list of
``Gate(kind, qubits, params)`` records; each side maps the kind NAME onto its
own gate table.

Conventions:
  * qubit q is bit q of the amplitude index (Eq. 2, stride 2^q);
  * ``qubits[0]`` is the least-significant axis of the gate's matrix index;
  * controlled kinds list controls first: CX(c, t), CP(c, t), CU(c, t),
    CCX(c0, c1, t).

Families and gate counts follow the paper's Table "benchmark circuits"
(PAPER.md P:L1930-1955); the closed forms m(n) are pinned against the printed
table in tests/golden/benchmark_gate_counts.json.

Seeds: numpy PCG64 with seed = 1000 * FAMILY_ID[family] + n; angles uniform
in [0, 2*pi).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Sequence, Tuple

import numpy as np

# Gate kind names accepted by both sides.
KINDS = (
    "H", "X", "Y", "Z", "S", "SDG", "T", "TDG", "RX", "RY", "RZ", "P", "U3",
    "CX", "CZ", "CP", "CCX", "SWAP", "CU",
)
ARITY = {k: 1 for k in KINDS[:13]}
ARITY.update({"CX": 2, "CZ": 2, "CP": 2, "SWAP": 2, "CU": 2, "CCX": 3})
NPARAMS = {k: 0 for k in KINDS}
NPARAMS.update({"RX": 1, "RY": 1, "RZ": 1, "P": 1, "CP": 1, "U3": 3, "CU": 4})

FAMILY_ID = {
    "qft": 1, "ghz": 2, "graphstate": 3, "qsvm": 4, "wstate": 5, "ising": 6,
    "su2random": 7, "random": 8,
}
FAMILIES = ("qft", "ghz", "graphstate", "qsvm", "wstate", "ising", "su2random")


@dataclass(frozen=True)
class Gate:
    kind: str
    qubits: Tuple[int, ...]
    params: Tuple[float, ...] = field(default_factory=tuple)

    def __post_init__(self):
        if self.kind not in ARITY:
            raise ValueError(f"unknown gate kind {self.kind}")
        if len(self.qubits) != ARITY[self.kind]:
            raise ValueError(f"{self.kind} takes {ARITY[self.kind]} qubits")
        if len(set(self.qubits)) != len(self.qubits):
            raise ValueError("duplicate operand")
        if len(self.params) != NPARAMS[self.kind]:
            raise ValueError(f"{self.kind} takes {NPARAMS[self.kind]} params")


@dataclass
class Circuit:
    n: int
    gates: List[Gate]
    name: str = ""
    seed: int = -1

    def __len__(self):
        return len(self.gates)


def _rng(family: str, n: int) -> Tuple[np.random.Generator, int]:
    seed = 1000 * FAMILY_ID[family] + n
    return np.random.default_rng(seed), seed


def _angle(rng) -> float:
    return float(rng.uniform(0.0, 2.0 * math.pi))


def qft(n: int) -> Circuit:
    """for target i: H(q_i); CP(pi/2^(j-i)) control q_j -> q_i for j > i.
    No terminal swaps.  m = n(n+1)/2."""
    g = []
    for i in range(n):
        g.append(Gate("H", (i,)))
        for j in range(i + 1, n):
            g.append(Gate("CP", (j, i), (math.pi / (1 << (j - i)),)))
    return Circuit(n, g, f"qft{n}")


def ghz(n: int) -> Circuit:
    """H(q0); CX(q_i -> q_{i+1}).  m = n."""
    g = [Gate("H", (0,))]
    for i in range(n - 1):
        g.append(Gate("CX", (i, i + 1)))
    return Circuit(n, g, f"ghz{n}")


def graphstate(n: int) -> Circuit:
    """H on all; CZ on the edges of a seeded random 2-regular graph (a random
    Hamiltonian cycle).  m = 2n."""
    rng, seed = _rng("graphstate", n)
    g = [Gate("H", (i,)) for i in range(n)]
    perm = [int(x) for x in rng.permutation(n)]
    for e in range(n):
        a, b = perm[e], perm[(e + 1) % n]
        g.append(Gate("CZ", (min(a, b), max(a, b))))
    return Circuit(n, g, f"graphstate{n}", seed)


def qsvm(n: int) -> Circuit:
    """ZZ feature map, 2 reps, linear entanglement.  m = 10n - 6."""
    rng, seed = _rng("qsvm", n)
    x = [_angle(rng) for _ in range(n)]
    g = []
    for _ in range(2):
        g += [Gate("H", (i,)) for i in range(n)]
        g += [Gate("P", (i,), (2.0 * x[i],)) for i in range(n)]
        for i in range(n - 1):
            phi = 2.0 * (math.pi - x[i]) * (math.pi - x[i + 1])
            g.append(Gate("CX", (i, i + 1)))
            g.append(Gate("P", (i + 1,), (phi,)))
            g.append(Gate("CX", (i, i + 1)))
    return Circuit(n, g, f"qsvm{n}", seed)


def wstate(n: int) -> Circuit:
    """X(q_{n-1}); for m=1..n-1 with i=n-m, j=n-m-1,
    theta=arccos(sqrt(1/(n-m+1))): RY(-theta) q_j, CZ(q_i,q_j), RY(theta) q_j;
    then CX(q_{k-1} -> q_k) for k = n-1..1.  m = 4n - 3."""
    g = [Gate("X", (n - 1,))]
    for m in range(1, n):
        i, j = n - m, n - m - 1
        th = math.acos(math.sqrt(1.0 / (n - m + 1)))
        g.append(Gate("RY", (j,), (-th,)))
        g.append(Gate("CZ", (j, i)))
        g.append(Gate("RY", (j,), (th,)))
    for k in range(n - 1, 0, -1):
        g.append(Gate("CX", (k - 1, k)))
    return Circuit(n, g, f"wstate{n}")


def ising(n: int) -> Circuit:
    """H all; 2 Trotter steps x [(n-1) x (CX, RZ, CX) + RX all + RZ all].
    m = 11n - 6."""
    rng, seed = _rng("ising", n)
    g = [Gate("H", (i,)) for i in range(n)]
    for _ in range(2):
        for i in range(n - 1):
            g.append(Gate("CX", (i, i + 1)))
            g.append(Gate("RZ", (i + 1,), (_angle(rng),)))
            g.append(Gate("CX", (i, i + 1)))
        g += [Gate("RX", (i,), (_angle(rng),)) for i in range(n)]
        g += [Gate("RZ", (i,), (_angle(rng),)) for i in range(n)]
    return Circuit(n, g, f"ising{n}", seed)


def su2random(n: int, reps: int = 3) -> Circuit:
    """EfficientSU2-like: (reps+1) layers of random U3 on every qubit,
    interleaved with `reps` full-entanglement CX blocks (i < j, row-major).
    m = n(3n+5)/2 for reps = 3."""
    rng, seed = _rng("su2random", n)
    g = []
    for r in range(reps + 1):
        g += [Gate("U3", (q,), (_angle(rng), _angle(rng), _angle(rng)))
              for q in range(n)]
        if r < reps:
            for i in range(n):
                for j in range(i + 1, n):
                    g.append(Gate("CX", (i, j)))
    return Circuit(n, g, f"su2random{n}", seed)


def random_circuit(n: int, m: int, seed: int, kinds: Sequence[str] = KINDS,
                   max_arity: int = 3) -> Circuit:
    """Uniformly random gates (kind, distinct qubits, angles) for parity and
    planner property tests."""
    rng = np.random.default_rng(1000 * FAMILY_ID["random"] + seed)
    ks = [k for k in kinds if ARITY[k] <= min(n, max_arity)]
    g = []
    for _ in range(m):
        k = ks[int(rng.integers(len(ks)))]
        qs = tuple(int(x) for x in rng.choice(n, size=ARITY[k], replace=False))
        ps = tuple(_angle(rng) for _ in range(NPARAMS[k]))
        g.append(Gate(k, qs, ps))
    return Circuit(n, g, f"random{n}_{m}_{seed}", seed)


def inverse(c: Circuit) -> Circuit:
    """The adjoint circuit C^dagger (mirror-circuit tests).
    Only parameter rewriting; no matrices."""
    inv = []
    for g in reversed(c.gates):
        k, p = g.kind, g.params
        if k in ("H", "X", "Y", "Z", "CX", "CZ", "SWAP", "CCX"):
            inv.append(g)
        elif k == "S":
            inv.append(Gate("SDG", g.qubits))
        elif k == "SDG":
            inv.append(Gate("S", g.qubits))
        elif k == "T":
            inv.append(Gate("TDG", g.qubits))
        elif k == "TDG":
            inv.append(Gate("T", g.qubits))
        elif k in ("RX", "RY", "RZ", "P", "CP"):
            inv.append(Gate(k, g.qubits, (-p[0],)))
        elif k == "U3":
            inv.append(Gate("U3", g.qubits, (-p[0], -p[2], -p[1])))
        elif k == "CU":
            inv.append(Gate("CU", g.qubits, (-p[0], -p[2], -p[1], -p[3])))
        else:
            raise ValueError(k)
    return Circuit(c.n, inv, c.name + "_inv", c.seed)


def mirror(c: Circuit) -> Circuit:
    """C followed by C^dagger: maps |0...0> back to |0...0>."""
    return Circuit(c.n, list(c.gates) + inverse(c).gates, c.name + "_mirror",
                   c.seed)


def prepend_basis(c: Circuit, x: int) -> Circuit:
    """Prepend X on the set bits of x so the circuit starts from |x>."""
    pre = [Gate("X", (q,)) for q in range(c.n) if (x >> q) & 1]
    return Circuit(c.n, pre + list(c.gates), f"{c.name}_from{x}", c.seed)


GENERATORS = {
    "qft": qft, "ghz": ghz, "graphstate": graphstate, "qsvm": qsvm,
    "wstate": wstate, "ising": ising, "su2random": su2random,
}


def make(family: str, n: int) -> Circuit:
    return GENERATORS[family](n)


def expected_gate_count(family: str, n: int) -> int:
    """Closed forms of the paper's table, SURVEY §8d."""
    return {
        "qft": n * (n + 1) // 2, "ghz": n, "graphstate": 2 * n,
        "qsvm": 10 * n - 6, "wstate": 4 * n - 3, "ising": 11 * n - 6,
        "su2random": n * (3 * n + 5) // 2,
    }[family]
