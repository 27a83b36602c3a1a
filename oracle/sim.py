"""O1: ctypes front-end of the C gate-at-a-time simulator (oracle/sv_oracle.c).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

``simulate(circuit)`` returns the 2^n complex128 state in logical order
(bit q of the index = qubit q).  Pinned by tests/test_oracle_sim.py:
GHZ / W / graph-state / QFT-of-basis-state closed forms, norm preservation,
full 2^n x 2^n unitaries against an independent Kronecker-product build,
mirror circuits, and agreement with the independent einsum simulator O1'.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import sys

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sv_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")          # 1 thread
_LIB_OMP = os.path.join(_HERE, "liboracle_omp.so")  # OpenMP over the host cores

# The oracle's own kind codes (order of the enum in sv_oracle.c).
KIND_CODE = {k: i for i, k in enumerate(
    ["H", "X", "Y", "Z", "S", "SDG", "T", "TDG", "RX", "RY", "RZ", "P", "U3",
     "CX", "CZ", "CP", "CCX", "SWAP", "CU"])}

_libs = {}


def _build_one(out, extra, force):
    if force or not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(_SRC):
        tmp = out + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-fPIC", "-shared", *extra,
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, out)
    return out


def build(force: bool = False) -> str:
    """Compile sv_oracle.c with plain gcc (-O2, no fast-math) twice: a
    single-threaded build and an OpenMP build of the same loops (the gate
    loop over amplitude groups split across host cores; identical
    arithmetic per amplitude, so both give bit-identical states)."""
    _build_one(_LIB_OMP, ["-fopenmp"], force)
    return _build_one(_LIB, [], force)


def lib(omp: bool = True):
    """The oracle library: the OpenMP build (default) or the 1-thread one."""
    key = bool(omp)
    if key not in _libs:
        build()
        L = ctypes.CDLL(_LIB_OMP if omp else _LIB)
        L.oracle_simulate.restype = ctypes.c_int
        L.oracle_simulate.argtypes = [
            ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        L.oracle_gate_matrix.restype = ctypes.c_int
        L.oracle_gate_matrix.argtypes = [ctypes.c_int, ctypes.c_void_p,
                                         ctypes.c_void_p, ctypes.c_void_p]
        L.oracle_norm2.restype = ctypes.c_double
        L.oracle_norm2.argtypes = [ctypes.c_void_p, ctypes.c_int]
        L.oracle_threads.restype = ctypes.c_int
        _libs[key] = L
    return _libs[key]


def threads(omp: bool = True) -> int:
    """Host threads the chosen build runs on."""
    return lib(omp).oracle_threads()


def encode(gates):
    m = len(gates)
    kinds = np.zeros(max(m, 1), dtype=np.int32)
    qubits = np.zeros((max(m, 1), 3), dtype=np.int32)
    params = np.zeros((max(m, 1), 4), dtype=np.float64)
    for i, g in enumerate(gates):
        kinds[i] = KIND_CODE[g.kind]
        qubits[i, :len(g.qubits)] = g.qubits
        params[i, :len(g.params)] = g.params
    return kinds, qubits, params


def simulate(circuit, init=None, gates=None, omp: bool = True) -> np.ndarray:
    """Run the circuit from |0...0> (or from `init`, copied) and return the
    final state vector (complex128, logical order).  omp=False runs the
    single-threaded build."""
    n = circuit.n
    gl = circuit.gates if gates is None else gates
    if init is None:
        psi = np.zeros(1 << n, dtype=np.complex128)
        zero = 1
    else:
        psi = np.array(init, dtype=np.complex128, copy=True)
        zero = 0
    kinds, qubits, params = encode(gl)
    rc = lib(omp).oracle_simulate(psi.ctypes.data, n, len(gl), kinds.ctypes.data,
                               qubits.ctypes.data, params.ctypes.data, zero)
    if rc != 0:
        raise RuntimeError(f"oracle_simulate failed rc={rc}")
    return psi


def gate_matrix(kind: str, params=()) -> np.ndarray:
    re = np.zeros(64)
    im = np.zeros(64)
    p = np.zeros(4)
    p[:len(params)] = params
    d = lib().oracle_gate_matrix(KIND_CODE[kind], p.ctypes.data, re.ctypes.data,
                                 im.ctypes.data)
    return (re[:d * d] + 1j * im[:d * d]).reshape(d, d)


def norm2(psi: np.ndarray, n: int) -> float:
    return lib().oracle_norm2(np.ascontiguousarray(psi).ctypes.data, n)


if __name__ == "__main__":  # pragma: no cover
    build(force="--force" in sys.argv)
    print(_LIB)
