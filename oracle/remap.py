"""O3: the inter-stage remap as a pure index permutation.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md Alg. Execute: ``Shard(shards, Q, P)`` permutes the
state vector so that the stage's local qubits are the low physical bits; the
permutation P is tracked.  Physical qubit p is bit p of the
physical index; the first L are local, the next R regional, the last G global
(Def. P:L1405-1417).  With a logical->physical map sigma (Fig. P:L1278,
"q_i[p_j]") and a mask of flipped physical bits (reading R14: an
anti-diagonal insular gate on a non-local qubit is a relabelling), logical
index x lives at physical index  phys(x) = (sum_q bit_q(x) << sigma[q]) ^ flip.

Pinned by: permutation properties (bijection, round trip = identity, the
multiset of amplitudes preserved bit-exactly) and Fig. qubit_remapping
 with L=R=G=1: swapping a local with a
regional qubit moves no amplitude across nodes; swapping a local with the
global qubit moves 4 of 8 amplitudes across nodes.
"""
from __future__ import annotations

import numpy as np


def phys_index(x: np.ndarray, sigma, flip: int = 0) -> np.ndarray:
    x = np.asarray(x, dtype=np.int64)
    p = np.zeros_like(x)
    for q, s in enumerate(sigma):
        p |= ((x >> q) & 1) << s
    return p ^ flip


def to_physical(logical_state: np.ndarray, sigma, flip: int = 0) -> np.ndarray:
    n = len(sigma)
    x = np.arange(1 << n, dtype=np.int64)
    out = np.empty_like(logical_state)
    out[phys_index(x, sigma, flip)] = logical_state
    return out


def to_logical(phys_state: np.ndarray, sigma, flip: int = 0) -> np.ndarray:
    n = len(sigma)
    x = np.arange(1 << n, dtype=np.int64)
    return phys_state[phys_index(x, sigma, flip)]


def remap(phys_state, sigma_old, flip_old, sigma_new, flip_new):
    """new[phys_new(x)] = old[phys_old(x)] for every logical x."""
    return to_physical(to_logical(phys_state, sigma_old, flip_old), sigma_new, flip_new)


def comm_counts(n: int, L: int, R: int, sigma_old, sigma_new):
    """Amplitudes whose node (physical bits >= L+R) changes = inter-node;
    same node but different shard (bits [L, L+R)) = intra-node."""
    x = np.arange(1 << n, dtype=np.int64)
    po = phys_index(x, sigma_old)
    pn = phys_index(x, sigma_new)
    node_o, node_n = po >> (L + R), pn >> (L + R)
    shard_o, shard_n = po >> L, pn >> L
    inter = int(np.sum(node_o != node_n))
    intra = int(np.sum((node_o == node_n) & (shard_o != shard_n)))
    return inter, intra
