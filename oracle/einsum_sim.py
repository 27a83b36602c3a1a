"""O1': an independent NumPy simulator on the 2 x ... x 2 tensor view.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md P:L709-714: "the state vector over n-qubits can be represented as a
tensor with n dimensions, each of which has a size of two ... Each quantum
gate can be considered as a linear transformation to the corresponding
dimensions, whose weights are given by the unitary matrix of the gate."

Written with ``np.tensordot`` on a reshaped tensor and the oracle's NumPy gate
table (oracle/gates.py), so it shares no indexing code with the C oracle O1.
Used for n <= 16 as a cross-check of O1.
"""
from __future__ import annotations

import numpy as np

from . import gates as G


def apply(psi_t: np.ndarray, n: int, u: np.ndarray, qubits) -> np.ndarray:
    k = len(qubits)
    # Tensor axes: numpy C-order reshape to (2,)*n puts qubit n-1 on axis 0,
    # qubit q on axis n-1-q.
    axes = [n - 1 - q for q in qubits]
    # Gate tensor: U[r, c] with r = sum_j r_j 2^j -> axes (r_{k-1} .. r_0, c_{k-1} .. c_0)
    ut = u.reshape((2,) * (2 * k))
    # contract gate input axes (c_j at position 2k-1-j) with state axes
    in_axes = [2 * k - 1 - j for j in range(k)]
    out = np.tensordot(ut, psi_t, axes=(in_axes, axes))
    # out axes: (r_{k-1}, ..., r_0, remaining state axes in order)
    remaining = [a for a in range(n) if a not in axes]
    # output gate axis r_j (position k-1-j) goes to state axis axes[j]
    perm_src = {}
    for j in range(k):
        perm_src[axes[j]] = k - 1 - j
    for i, a in enumerate(remaining):
        perm_src[a] = k + i
    return np.transpose(out, [perm_src[a] for a in range(n)])


def simulate(circuit, init=None) -> np.ndarray:
    n = circuit.n
    if n > 16:
        raise ValueError("O1' is for n <= 16")
    if init is None:
        psi = np.zeros(1 << n, dtype=np.complex128)
        psi[0] = 1.0
    else:
        psi = np.array(init, dtype=np.complex128)
    t = psi.reshape((2,) * n)
    for g in circuit.gates:
        t = apply(t, n, G.matrix(g.kind, g.params), g.qubits)
    return np.ascontiguousarray(t).reshape(-1)
