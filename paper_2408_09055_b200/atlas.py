"""Thin ctypes binding of include/atlas.h (argument marshalling only).

Every step of the simulation runs inside libatlas_b200.so (host planner in
C++, device path in sm_100a CUDA).  There is no Python or CPU fallback: if
the shared library is missing or a call fails, an AtlasError is raised.
"""
from __future__ import annotations

import ctypes
import json
import os
from typing import Iterable, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libatlas_b200.so")

C128, C64 = 0, 1

KIND = {k: i for i, k in enumerate(
    ["H", "X", "Y", "Z", "S", "SDG", "T", "TDG", "RX", "RY", "RZ", "P", "U3",
     "CX", "CZ", "CP", "CCX", "SWAP", "CU"])}

STATUS = {0: "OK", 1: "E_INVALID", 2: "E_UNSUPPORTED", 3: "E_INFEASIBLE", 4: "E_BUDGET",
          5: "E_OOM", 6: "E_CUDA", 7: "E_NCCL", 8: "E_ORDER"}

LAUNCH_KIND = {0: "init", 1: "fused", 2: "shm", 3: "pack", 4: "exchange", 5: "scale", 6: "h2d", 7: "d2h"}

# exported symbols (include/atlas.h); the CPU test checks each is present
SYMBOLS = [
    "atlas_create", "atlas_load_circuit", "atlas_plan", "atlas_run", "atlas_get_state",
    "atlas_set_state", "atlas_destroy", "atlas_last_error", "atlas_set_option_int",
    "atlas_set_option_str", "atlas_bind_buffers", "atlas_set_stream", "atlas_nccl_unique_id",
    "atlas_get_plan_json", "atlas_plan_stats", "atlas_get_launches", "atlas_remap_schedule",
    "atlas_get_jit_source",
]


class AtlasError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class Xfer(ctypes.Structure):
    _fields_ = [("peer", ctypes.c_int32), ("kind", ctypes.c_int32),
                ("src_off", ctypes.c_uint64), ("dst_off", ctypes.c_uint64),
                ("bytes", ctypes.c_uint64)]


XFER_KIND = {0: "send", 1: "recv", 2: "local"}


class Gate(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_uint32), ("nq", ctypes.c_uint32),
                ("q", ctypes.c_uint32 * 3), ("pad_", ctypes.c_uint32),
                ("p", ctypes.c_double * 4)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise AtlasError(6, f"{LIB_PATH} not built (run python -m paper_2408_09055_b200.build)")
        L = ctypes.CDLL(LIB_PATH)
        vp, sz, i32, i64, u64, dbl = (ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int,
                                      ctypes.c_int64, ctypes.c_uint64, ctypes.c_double)
        sig = {
            "atlas_create": [i32, i32, i32, i32, vp, ctypes.POINTER(vp)],
            "atlas_load_circuit": [vp, vp, sz],
            "atlas_plan": [vp, i32, dbl],
            "atlas_run": [vp],
            "atlas_get_state": [vp, vp, u64, u64],
            "atlas_set_state": [vp, vp, u64, u64],
            "atlas_set_option_int": [vp, ctypes.c_char_p, i64],
            "atlas_set_option_str": [vp, ctypes.c_char_p, ctypes.c_char_p],
            "atlas_bind_buffers": [vp, vp, vp, u64],
            "atlas_set_stream": [vp, vp],
            "atlas_nccl_unique_id": [vp],
            "atlas_get_plan_json": [vp, vp, sz, ctypes.POINTER(sz)],
            "atlas_plan_stats": [vp, vp, i32],
            "atlas_get_launches": [vp, vp, vp, vp, i32, ctypes.POINTER(i32)],
            "atlas_remap_schedule": [vp, i32, vp, i32, ctypes.POINTER(i32)],
            "atlas_get_jit_source": [vp, i32, i32, vp, sz, ctypes.POINTER(sz)],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = ctypes.c_int
        L.atlas_destroy.argtypes = [vp]
        L.atlas_destroy.restype = None
        L.atlas_last_error.argtypes = []
        L.atlas_last_error.restype = ctypes.c_char_p
        _lib = L
    return _lib


def _check(st):
    if st != 0:
        msg = lib().atlas_last_error()
        raise AtlasError(st, msg.decode() if msg else "")


def encode_gates(gates) -> ctypes.Array:
    """gates: iterable of objects with .kind (name), .qubits, .params."""
    gl = list(gates)
    arr = (Gate * max(len(gl), 1))()
    for i, g in enumerate(gl):
        a = arr[i]
        a.kind = KIND[g.kind]
        a.nq = len(g.qubits)
        for j, q in enumerate(g.qubits):
            a.q[j] = q
        for j, p in enumerate(g.params):
            a.p[j] = p
    return arr, len(gl)


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().atlas_nccl_unique_id(buf))
    return buf.raw


class Simulator:
    """One atlas_ctx.  Mirrors the C calls one to one."""

    def __init__(self, n: int, dtype: int = C128, world: int = 1, rank: int = 0,
                 nccl_uid: Optional[bytes] = None, **options):
        self.n, self.dtype, self.world, self.rank = n, dtype, world, rank
        self._ctx = ctypes.c_void_p()
        uid = ctypes.create_string_buffer(nccl_uid, 128) if nccl_uid else None
        _check(lib().atlas_create(n, dtype, world, rank, uid, ctypes.byref(self._ctx)))
        for k, v in options.items():
            self.set_option(k, v)

    def close(self):
        if self._ctx:
            lib().atlas_destroy(self._ctx)
            self._ctx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def np_dtype(self):
        return np.complex128 if self.dtype == C128 else np.complex64

    def set_option(self, key: str, value):
        if isinstance(value, str):
            _check(lib().atlas_set_option_str(self._ctx, key.encode(), value.encode()))
        else:
            _check(lib().atlas_set_option_int(self._ctx, key.encode(), int(value)))

    def load_circuit(self, gates):
        arr, m = encode_gates(gates)
        _check(lib().atlas_load_circuit(self._ctx, arr, m))

    def plan(self, s_max: int = 16, c: float = 3.0):
        _check(lib().atlas_plan(self._ctx, s_max, c))

    def run(self):
        _check(lib().atlas_run(self._ctx))

    def get_state(self, first: int = 0, count: Optional[int] = None, out=None) -> np.ndarray:
        if count is None:
            count = (1 << self.n) - first
        if out is None:
            out = np.zeros(count, dtype=self.np_dtype)
        _check(lib().atlas_get_state(self._ctx, out.ctypes.data, first, count))
        return out

    def get_state_into(self, ptr: int, first: int, count: int):
        """Copy into caller-owned host memory at address ptr (e.g. pinned)."""
        _check(lib().atlas_get_state(self._ctx, ptr, first, count))

    def set_state_from(self, ptr: int, first: int, count: int):
        """Copy from caller-owned host memory at address ptr (e.g. pinned)."""
        _check(lib().atlas_set_state(self._ctx, ptr, first, count))

    def set_state(self, psi: np.ndarray, first: int = 0):
        a = np.ascontiguousarray(psi, dtype=self.np_dtype)
        _check(lib().atlas_set_state(self._ctx, a.ctypes.data, first, len(a)))

    def bind_buffers(self, state_ptr: int, scratch_ptr: int, nbytes: int):
        _check(lib().atlas_bind_buffers(self._ctx, state_ptr, scratch_ptr, nbytes))

    def set_stream(self, stream_ptr: int):
        _check(lib().atlas_set_stream(self._ctx, stream_ptr))

    def plan_json(self) -> dict:
        n = ctypes.c_size_t()
        _check(lib().atlas_get_plan_json(self._ctx, None, 0, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(n.value + 1)
        _check(lib().atlas_get_plan_json(self._ctx, buf, n.value + 1, ctypes.byref(n)))
        return json.loads(buf.value.decode())

    def plan_stats(self) -> dict:
        v = (ctypes.c_int64 * 14)()
        _check(lib().atlas_plan_stats(self._ctx, v, 14))
        keys = ["stages", "staging_cost_x1000", "kernels", "fusion_kernels", "shm_kernels",
                "kernel_cost", "remaps", "plan_us", "staging_exact", "L", "G",
                "launches_per_run", "jit_us", "stage_us"]
        return dict(zip(keys, list(v)))

    def jit_source(self, index: int, slot: int = 0) -> str:
        """CUDA source of the plan-specialised kernel of shared-memory launch
        `index` of simulated rank `slot` (host-only)."""
        n = ctypes.c_size_t()
        _check(lib().atlas_get_jit_source(self._ctx, slot, index, None, 0, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(n.value + 1)
        _check(lib().atlas_get_jit_source(self._ctx, slot, index, buf, n.value + 1,
                                          ctypes.byref(n)))
        return buf.value.decode()

    def remap_schedule(self, stage: int):
        """This rank's transfers of the remap before `stage`:
        [(kind, peer, src_off, dst_off, bytes)] (host-only)."""
        cnt = ctypes.c_int()
        _check(lib().atlas_remap_schedule(self._ctx, stage, None, 0, ctypes.byref(cnt)))
        buf = (Xfer * max(cnt.value, 1))()
        _check(lib().atlas_remap_schedule(self._ctx, stage, buf, cnt.value, ctypes.byref(cnt)))
        return [(XFER_KIND[x.kind], x.peer, x.src_off, x.dst_off, x.bytes)
                for x in buf[:cnt.value]]

    def launches(self):
        cnt = ctypes.c_int()
        _check(lib().atlas_get_launches(self._ctx, None, None, None, 0, ctypes.byref(cnt)))
        n = cnt.value
        ms = (ctypes.c_float * max(n, 1))()
        kd = (ctypes.c_int32 * max(n, 1))()
        by = (ctypes.c_int64 * max(n, 1))()
        _check(lib().atlas_get_launches(self._ctx, ms, kd, by, n, ctypes.byref(cnt)))
        return [(LAUNCH_KIND[kd[i]], float(ms[i]), int(by[i])) for i in range(n)]


def simulate(circuit, dtype: int = C128, s_max: int = 16, c: float = 3.0, world: int = 1,
             **options) -> np.ndarray:
    """Convenience: plan + run one circuit (world=1, or virtual world on one GPU)."""
    if world > 1:
        options.setdefault("virtual_world", 1)
    with Simulator(circuit.n, dtype, world, 0, **options) as s:
        s.load_circuit(circuit.gates)
        s.plan(s_max, c)
        s.run()
        return s.get_state()
