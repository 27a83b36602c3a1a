"""The oracle's own gate table (NumPy) and insularity *by definition*.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Matrices: textbook / OpenQASM 2 definitions; operand
qubits[0] is the least-significant bit of the matrix index.
This table is written independently of oracle/sv_oracle.c (a second copy in a
different language, used by the einsum simulator O1') so that a typo in one is
caught by the O1 == O1' pin.

Insularity (Def. "Insular Qubit") is evaluated from the
matrix, not from a kind table:
  * 1-qubit gate: insular iff U is diagonal or anti-diagonal (|entry| < 1e-12
    counts as zero);
  * multi-qubit gate: operand q is a *control* iff U never mixes q=0 with q=1
    and acts as the identity on the q=0 subspace; all controls are insular.
    The footnote's symmetric gates (CZ, CP: "any qubit can be chosen as the
    control") then come out with every operand insular without a special case.
Pinned by tests/test_oracle_planner.py against the paper's own examples
(Z insular, CX control-only, CZ both, H none: SPEC S:L84-87 quoting the Def.).
"""
from __future__ import annotations

import cmath
import math

import numpy as np

TOL = 1e-12


def matrix(kind: str, params=()) -> np.ndarray:
    p = list(params)
    r2 = 1.0 / math.sqrt(2.0)
    if kind == "H":
        return np.array([[r2, r2], [r2, -r2]], dtype=complex)
    if kind == "X":
        return np.array([[0, 1], [1, 0]], dtype=complex)
    if kind == "Y":
        return np.array([[0, -1j], [1j, 0]], dtype=complex)
    if kind == "Z":
        return np.diag([1, -1]).astype(complex)
    if kind == "S":
        return np.diag([1, 1j])
    if kind == "SDG":
        return np.diag([1, -1j])
    if kind == "T":
        return np.diag([1, cmath.exp(1j * math.pi / 4)])
    if kind == "TDG":
        return np.diag([1, cmath.exp(-1j * math.pi / 4)])
    if kind == "RX":
        c, s = math.cos(p[0] / 2), math.sin(p[0] / 2)
        return np.array([[c, -1j * s], [-1j * s, c]])
    if kind == "RY":
        c, s = math.cos(p[0] / 2), math.sin(p[0] / 2)
        return np.array([[c, -s], [s, c]], dtype=complex)
    if kind == "RZ":
        return np.diag([cmath.exp(-1j * p[0] / 2), cmath.exp(1j * p[0] / 2)])
    if kind == "P":
        return np.diag([1, cmath.exp(1j * p[0])])
    if kind == "U3":
        t, ph, la = p
        c, s = math.cos(t / 2), math.sin(t / 2)
        return np.array([[c, -cmath.exp(1j * la) * s],
                         [cmath.exp(1j * ph) * s, cmath.exp(1j * (ph + la)) * c]])
    if kind in ("CX", "CZ", "CP", "CU"):
        # controlled-V with control = index bit 0, target = index bit 1:
        # |c=0> block is identity; |c=1> block is V on the target.
        if kind == "CX":
            v = matrix("X")
        elif kind == "CZ":
            v = matrix("Z")
        elif kind == "CP":
            v = matrix("P", p[:1])
        else:
            v = cmath.exp(1j * p[3]) * matrix("U3", p[:3])
        u = np.zeros((4, 4), dtype=complex)
        for t_out in range(2):
            for t_in in range(2):
                u[0 + 2 * t_out, 0 + 2 * t_in] = 1.0 if t_out == t_in else 0.0
                u[1 + 2 * t_out, 1 + 2 * t_in] = v[t_out, t_in]
        return u
    if kind == "SWAP":
        u = np.zeros((4, 4), dtype=complex)
        for b0 in range(2):
            for b1 in range(2):
                u[b1 + 2 * b0, b0 + 2 * b1] = 1.0
        return u
    if kind == "CCX":
        u = np.eye(8, dtype=complex)
        u[[3, 7], :] = u[[7, 3], :]
        return u
    raise ValueError(kind)


def arity(kind: str) -> int:
    return int(round(math.log2(matrix(kind, _dummy_params(kind)).shape[0])))


def _dummy_params(kind):
    return {"RX": (0.3,), "RY": (0.3,), "RZ": (0.3,), "P": (0.3,), "CP": (0.3,),
            "U3": (0.3, 0.2, 0.1), "CU": (0.3, 0.2, 0.1, 0.05)}.get(kind, ())


def _is_control(u: np.ndarray, j: int, k: int) -> bool:
    d = 1 << k
    for r in range(d):
        for c in range(d):
            if ((r >> j) & 1) != ((c >> j) & 1) and abs(u[r, c]) > TOL:
                return False  # mixes q=0 and q=1
            if not ((r >> j) & 1) and not ((c >> j) & 1):
                want = 1.0 if r == c else 0.0
                if abs(u[r, c] - want) > TOL:
                    return False  # not the identity on the q=0 block
    return True


def insular_kind(kind: str, params=()) -> tuple:
    """Per operand: 'diag', 'anti' or None (non-insular).

    1-qubit: 'diag' if diagonal, 'anti' if anti-diagonal (Def. P:L1432-1434).
    Multi-qubit: controls are 'diag' (a control is a diagonal structure on its
    qubit), everything else None."""
    u = matrix(kind, params)
    k = int(round(math.log2(u.shape[0])))
    if k == 1:
        if abs(u[0, 1]) < TOL and abs(u[1, 0]) < TOL:
            return ("diag",)
        if abs(u[0, 0]) < TOL and abs(u[1, 1]) < TOL:
            return ("anti",)
        return (None,)
    return tuple("diag" if _is_control(u, j, k) else None for j in range(k))


def insular_qubits(kind: str, params=()) -> set:
    """Operand positions that are insular (SPEC insular_qubits)."""
    return {j for j, t in enumerate(insular_kind(kind, params)) if t is not None}
