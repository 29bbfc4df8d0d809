"""ORACLE -- test infrastructure only.

ctypes wrapper around ``oracle/qsim_oracle.c``, the plain CPU fp64
state-vector simulator written from PAPER.md (arXiv:1805.04708).  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  It shares no code with the
CUDA path (``paper_1805_04708_b200``), and the CUDA path never imports it.

Each wrapper names the PAPER.md passage its C function follows; see the C
file's header for the conventions and DESIGN.md for the readings.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "qsim_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

_dp = ctypes.POINTER(ctypes.c_double)
_i8p = ctypes.POINTER(ctypes.c_int8)
_i32p = ctypes.POINTER(ctypes.c_int32)


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C, OpenMP over the outer loop)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        L = _lib
        L.oracle_e_init.argtypes = [_dp, ctypes.c_int]
        L.oracle_e_apply.argtypes = [_dp, ctypes.c_int, _dp, ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.c_int]
        L.oracle_e_swap.argtypes = [_dp, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.oracle_e_run.argtypes = [_dp, ctypes.c_int, ctypes.c_int64, _i32p, _i32p, _i32p, _i32p, _i32p, _dp]
        L.oracle_e_norm2.argtypes = [_dp, ctypes.c_int]
        L.oracle_e_norm2.restype = ctypes.c_double
        L.oracle_e_expectations.argtypes = [_dp, ctypes.c_int, _dp]
        L.oracle_e_probabilities.argtypes = [_dp, ctypes.c_int, _dp]
        L.oracle_e_measure.argtypes = [_dp, ctypes.c_int, ctypes.c_int, ctypes.c_double, _dp]
        L.oracle_e_shorbox.argtypes = [_dp, ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64]
        L.oracle_e_sample.argtypes = [_dp, ctypes.c_int, _dp, ctypes.c_int64, ctypes.POINTER(ctypes.c_uint64)]
        L.oracle_e_project.argtypes = [_dp, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.oracle_a_decode.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double, _dp, _dp]
        L.oracle_a_encode.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                      ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]
        L.oracle_a_bounds.argtypes = [_dp, ctypes.c_uint64, _dp, _dp]
        L.oracle_a_init.argtypes = [_i8p, ctypes.c_int, _dp, _dp]
        L.oracle_a_decode_state.argtypes = [_i8p, ctypes.c_int, ctypes.c_double, ctypes.c_double, _dp]
        L.oracle_a_encode_state.argtypes = [_dp, ctypes.c_int, _i8p, _dp, _dp]
        L.oracle_a_apply.argtypes = [_i8p, ctypes.c_int, _dp, _dp, _dp, ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                                     ctypes.c_int, _dp]
        L.oracle_a_run.argtypes = [_i8p, ctypes.c_int, _dp, _dp, ctypes.c_int64, _i32p, _i32p, _i32p, _i32p, _i32p,
                                   _dp, _dp]
        L.oracle_a_apply_lazy.argtypes = L.oracle_a_apply.argtypes
        L.oracle_a_apply_lazy.restype = ctypes.c_int
        L.oracle_a_run_lazy.argtypes = L.oracle_a_run.argtypes
        L.oracle_a_run_lazy.restype = ctypes.c_int64
        L.oracle_num_threads.restype = ctypes.c_int
        L.oracle_set_num_threads.argtypes = [ctypes.c_int]
        L.oracle_set_num_threads.restype = None
    return _lib


def _ptr(arr, t):
    return arr.ctypes.data_as(t)


def _c128(a: np.ndarray) -> np.ndarray:
    assert a.dtype == np.complex128 and a.flags.c_contiguous
    return a


# ----------------------------------------------------------------------------- E


def e_init(n: int) -> np.ndarray:
    """|0...0> (Eq. appa0)."""
    a = np.empty(1 << n, dtype=np.complex128)
    lib().oracle_e_init(_ptr(a.view(np.float64), _dp), n)
    return a


def e_apply(a: np.ndarray, n: int, u, target: int, controls=()) -> np.ndarray:
    """Eq. NUM2 with controls, in place."""
    _c128(a)
    u8 = np.ascontiguousarray(np.asarray(u, dtype=np.complex128).reshape(2, 2)).view(np.float64).reshape(8)
    c = (ctypes.c_int * 2)(*(list(controls) + [0, 0])[:2])
    lib().oracle_e_apply(_ptr(a.view(np.float64), _dp), n, _ptr(u8, _dp), target, c, len(controls))
    return a


def e_swap(a: np.ndarray, n: int, q1: int, q2: int) -> np.ndarray:
    _c128(a)
    lib().oracle_e_swap(_ptr(a.view(np.float64), _dp), n, q1, q2)
    return a


def e_run(a: np.ndarray, n: int, circuit) -> np.ndarray:
    """Apply a circuit (qsim_inputs.Circuit arrays) in order."""
    _c128(a)
    g = circuit
    lib().oracle_e_run(_ptr(a.view(np.float64), _dp), n, len(g.kind), _ptr(g.kind, _i32p), _ptr(g.target, _i32p),
                       _ptr(g.target2, _i32p), _ptr(g.nctrl, _i32p), _ptr(g.ctrl, _i32p), _ptr(g.u, _dp))
    return a


def e_simulate(n: int, circuit) -> np.ndarray:
    return e_run(e_init(n), n, circuit)


def e_norm2(a: np.ndarray, n: int) -> float:
    return lib().oracle_e_norm2(_ptr(_c128(a).view(np.float64), _dp), n)


def e_expectations(a: np.ndarray, n: int) -> np.ndarray:
    """BEGIN MEASUREMENT: rows (<Qx>, <Qy>, <Qz>) per qubit."""
    q = np.empty(3 * n, dtype=np.float64)
    lib().oracle_e_expectations(_ptr(_c128(a).view(np.float64), _dp), n, _ptr(q, _dp))
    return q.reshape(n, 3)


def e_probabilities(a: np.ndarray, n: int) -> np.ndarray:
    p = np.empty(n, dtype=np.float64)
    lib().oracle_e_probabilities(_ptr(_c128(a).view(np.float64), _dp), n, _ptr(p, _dp))
    return p


def e_measure(a: np.ndarray, n: int, qubit: int, u_draw: float):
    """M with a caller-drawn uniform u; returns (outcome, p0)."""
    p0 = ctypes.c_double(0.0)
    out = lib().oracle_e_measure(_ptr(_c128(a).view(np.float64), _dp), n, qubit, float(u_draw), ctypes.byref(p0))
    return out, p0.value


def e_shorbox(n: int, nx: int, G: int, y: int) -> np.ndarray:
    """SHORBOX: 2^{-nx/2} sum_x |x>|y^x mod G>, x on qubits 0..nx-1."""
    a = np.empty(1 << n, dtype=np.complex128)
    lib().oracle_e_shorbox(_ptr(a.view(np.float64), _dp), n, nx, G, y)
    return a


def e_sample(a: np.ndarray, n: int, u) -> np.ndarray:
    """GENERATE EVENTS: inverse-CDF indices for caller-drawn u in [0,1)."""
    u = np.ascontiguousarray(u, dtype=np.float64)
    out = np.empty(u.size, dtype=np.uint64)
    lib().oracle_e_sample(_ptr(_c128(a).view(np.float64), _dp), n, _ptr(u, _dp), u.size,
                          out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
    return out


def e_project(a: np.ndarray, n: int, qubit: int, value: int) -> int:
    """CLEAR / SET: project onto |value> of qubit, renormalise; -5 on zero norm."""
    return lib().oracle_e_project(_ptr(_c128(a).view(np.float64), _dp), n, qubit, value)


# ----------------------------------------------------------------------------- A


def a_decode(b0: int, b1: int, r0: float, r1: float) -> complex:
    """PAPER.md:449-453."""
    zr, zi = ctypes.c_double(), ctypes.c_double()
    lib().oracle_a_decode(int(b0), int(b1), float(r0), float(r1), ctypes.byref(zr), ctypes.byref(zi))
    return complex(zr.value, zi.value)


def a_encode(z: complex, r0: float, r1: float):
    b0, b1 = ctypes.c_int(), ctypes.c_int()
    lib().oracle_a_encode(float(z.real), float(z.imag), float(r0), float(r1), ctypes.byref(b0), ctypes.byref(b1))
    return b0.value, b1.value


def a_bounds(z: np.ndarray):
    r0, r1 = ctypes.c_double(), ctypes.c_double()
    lib().oracle_a_bounds(_ptr(_c128(z).view(np.float64), _dp), z.size, ctypes.byref(r0), ctypes.byref(r1))
    return r0.value, r1.value


class AState:
    """A-variant state: int8 codes interleaved (b0, b1) per amplitude + bounds."""

    def __init__(self, n: int, codes: np.ndarray | None = None, r0: float = 0.5, r1: float = 0.5):
        self.n = n
        if codes is None:
            self.codes = np.empty(2 << n, dtype=np.int8)
            r0c, r1c = ctypes.c_double(), ctypes.c_double()
            lib().oracle_a_init(_ptr(self.codes, _i8p), n, ctypes.byref(r0c), ctypes.byref(r1c))
            self.r0, self.r1 = r0c.value, r1c.value
        else:
            self.codes = np.ascontiguousarray(codes, dtype=np.int8).reshape(2 << n).copy()
            self.r0, self.r1 = float(r0), float(r1)
        self._work = None

    def work(self):
        if self._work is None:
            self._work = np.empty(2 << self.n, dtype=np.float64)
        return self._work

    def decoded(self) -> np.ndarray:
        z = np.empty(1 << self.n, dtype=np.complex128)
        lib().oracle_a_decode_state(_ptr(self.codes, _i8p), self.n, self.r0, self.r1, _ptr(z.view(np.float64), _dp))
        return z

    def encode_from(self, z: np.ndarray):
        r0c, r1c = ctypes.c_double(), ctypes.c_double()
        lib().oracle_a_encode_state(_ptr(_c128(z).view(np.float64), _dp), self.n, _ptr(self.codes, _i8p),
                                    ctypes.byref(r0c), ctypes.byref(r1c))
        self.r0, self.r1 = r0c.value, r1c.value

    def apply(self, u, target: int, controls=()):
        u8 = np.ascontiguousarray(np.asarray(u, dtype=np.complex128).reshape(2, 2)).view(np.float64).reshape(8)
        c = (ctypes.c_int * 2)(*(list(controls) + [0, 0])[:2])
        r0c, r1c = ctypes.c_double(self.r0), ctypes.c_double(self.r1)
        lib().oracle_a_apply(_ptr(self.codes, _i8p), self.n, ctypes.byref(r0c), ctypes.byref(r1c), _ptr(u8, _dp),
                             target, c, len(controls), _ptr(self.work(), _dp))
        self.r0, self.r1 = r0c.value, r1c.value

    def apply_lazy(self, u, target: int, controls=()) -> bool:
        """One gate under the lazy-bounds policy (reading R-A25); True if it rescaled."""
        u8 = np.ascontiguousarray(np.asarray(u, dtype=np.complex128).reshape(2, 2)).view(np.float64).reshape(8)
        c = (ctypes.c_int * 2)(*(list(controls) + [0, 0])[:2])
        r0c, r1c = ctypes.c_double(self.r0), ctypes.c_double(self.r1)
        rs = lib().oracle_a_apply_lazy(_ptr(self.codes, _i8p), self.n, ctypes.byref(r0c), ctypes.byref(r1c),
                                       _ptr(u8, _dp), target, c, len(controls), _ptr(self.work(), _dp))
        self.r0, self.r1 = r0c.value, r1c.value
        return bool(rs)

    def run_lazy(self, circuit) -> int:
        """A circuit under the lazy-bounds policy; returns the number of rescales."""
        g = circuit
        r0c, r1c = ctypes.c_double(self.r0), ctypes.c_double(self.r1)
        rs = lib().oracle_a_run_lazy(_ptr(self.codes, _i8p), self.n, ctypes.byref(r0c), ctypes.byref(r1c),
                                     len(g.kind), _ptr(g.kind, _i32p), _ptr(g.target, _i32p), _ptr(g.target2, _i32p),
                                     _ptr(g.nctrl, _i32p), _ptr(g.ctrl, _i32p), _ptr(g.u, _dp), _ptr(self.work(), _dp))
        self.r0, self.r1 = r0c.value, r1c.value
        return int(rs)

    def run(self, circuit):
        g = circuit
        r0c, r1c = ctypes.c_double(self.r0), ctypes.c_double(self.r1)
        lib().oracle_a_run(_ptr(self.codes, _i8p), self.n, ctypes.byref(r0c), ctypes.byref(r1c), len(g.kind),
                           _ptr(g.kind, _i32p), _ptr(g.target, _i32p), _ptr(g.target2, _i32p), _ptr(g.nctrl, _i32p),
                           _ptr(g.ctrl, _i32p), _ptr(g.u, _dp), _ptr(self.work(), _dp))
        self.r0, self.r1 = r0c.value, r1c.value
        return self


def num_threads() -> int:
    return lib().oracle_num_threads()


def set_num_threads(n: int) -> None:
    """OpenMP thread count of the oracle's loops (timing only; results unchanged)."""
    lib().oracle_set_num_threads(int(n))
