"""paper_1805_04708_b200 -- B200-native JUQCS hot path (arXiv:1805.04708).

Thin ctypes binding over ``libqsim.so`` (the C-ABI declared in
``include/qsim.h``).  Argument marshalling only: every step of the path runs
in the library's sm_100a kernels.  There is no CPU fallback: importing this
package fails loudly when ``libqsim.so`` is missing, and every compute call
raises ``QsimError`` (code QSIM_ECUDA) when no GPU is usable.

Function names mirror the C-ABI (``qsim_create``, ``qsim_apply_gate``,
``qsim_apply_circuit``, ``qsim_probabilities``, ``qsim_measure``,
``qsim_get_amplitudes`` ...); ``State`` is a convenience wrapper around them.
"""
from __future__ import annotations

import atexit
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libqsim.so")

QSIM_OK = 0
QSIM_EINVAL = -1
QSIM_ENOMEM = -2
QSIM_ECUDA = -3
QSIM_ECOMM = -4
QSIM_EZERONORM = -5
QSIM_ENOTUNITARY = -6
QSIM_EUNSUPPORTED = -7

ENC_FP64 = 0
ENC_ADAPTIVE2 = 1
TRANSPORT_LOCAL = 0
TRANSPORT_NCCL = 1
TRANSPORT_DEVICES = 2
A_POLICY_EXACT = 0
A_POLICY_LAZY = 1
A_POLICY_FP32 = 2
GATE_U = 0
GATE_SWAP = 1
OP_EXCHANGE = 0
OP_GATE = 1
OP_RELABEL = 2  # permutation gate on global bits: shard relabelling, no data movement
OP_REMAP = 3  # one (g, l) pair of a multi-bit all-to-all remap (consecutive ops, same gate_index)


class QsimError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"qsim error {code}: {msg}")
        self.code = code


class qsim_gate(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("target", ctypes.c_int32), ("target2", ctypes.c_int32),
                ("ncontrols", ctypes.c_int32), ("controls", ctypes.c_int32 * 2), ("u", ctypes.c_double * 8)]


class qsim_config(ctypes.Structure):
    _fields_ = [("n_qubits", ctypes.c_int32), ("encoding", ctypes.c_int32), ("nshards", ctypes.c_int32),
                ("transport", ctypes.c_int32), ("rank", ctypes.c_int32), ("device", ctypes.c_int32),
                ("nccl_id", ctypes.c_void_p), ("chunk_bytes", ctypes.c_int64), ("fuse", ctypes.c_int32),
                ("a_policy", ctypes.c_int32)]


class qsim_stats(ctypes.Structure):
    _fields_ = [("gates", ctypes.c_int64), ("kernels", ctypes.c_int64), ("sweeps", ctypes.c_int64),
                ("passes", ctypes.c_int64), ("fused_gates", ctypes.c_int64), ("exchanges", ctypes.c_int64),
                ("hbm_bytes", ctypes.c_double), ("gate_bytes", ctypes.c_double),
                ("exchange_bytes", ctypes.c_double), ("stages", ctypes.c_int64), ("jit_passes", ctypes.c_int64),
                ("a_rescales", ctypes.c_int64), ("a_dense", ctypes.c_int64)]


class qsim_kernel_profile(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("pad", ctypes.c_int32), ("launches", ctypes.c_int64),
                ("ms", ctypes.c_double), ("bytes", ctypes.c_double), ("flops", ctypes.c_double)]


KERNEL_NAMES = {0: "pass_e", 1: "sweep_e", 2: "xchg", 3: "a_bounds", 4: "a_apply", 5: "a_fast"}


class qsim_plan_op(ctypes.Structure):
    _fields_ = [("type", ctypes.c_int32), ("g", ctypes.c_int32), ("l", ctypes.c_int32), ("cls", ctypes.c_int32),
                ("ncontrols", ctypes.c_int32), ("controls", ctypes.c_int32 * 2), ("gate_index", ctypes.c_int32)]


assert ctypes.sizeof(qsim_gate) == 88

# every symbol include/qsim.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "qsim_create", "qsim_create_ex", "qsim_destroy", "qsim_nccl_unique_id", "qsim_apply_gate", "qsim_apply_swap",
    "qsim_apply_circuit", "qsim_norm", "qsim_probabilities", "qsim_expectations", "qsim_measure", "qsim_measure_u",
    "qsim_get_amplitudes", "qsim_get_state", "qsim_set_state", "qsim_get_codes", "qsim_set_codes", "qsim_sync",
    "qsim_project", "qsim_sample", "qsim_prepare_shorbox", "qsim_stream", "qsim_get_stats", "qsim_reset", "qsim_reset_basis", "qsim_profile", "qsim_profile_read", "qsim_reset_stats", "qsim_get_qubit_map", "qsim_last_error",
    "qsim_plan_create", "qsim_plan_num_ops", "qsim_plan_get_op", "qsim_plan_final_map", "qsim_plan_destroy",
    "qsim_aux_amplitudes", "qsim_aux_num_vars", "qsim_set_qubit_map",
    "qsim_asm_parse", "qsim_asm_info", "qsim_asm_get_op", "qsim_asm_destroy", "qsim_asm_run",
    "qsim_asm_result_get", "qsim_asm_result_destroy",
    "qsim_overlap", "qsim_apply_circuit_persistent", "qsim_magnitude_range", "qsim_get_bounds", "qsim_apply_matrix", "qsim_jit_sync", "qsim_jit_shutdown", "qsim_graph_begin", "qsim_graph_end", "qsim_graph_launch", "qsim_graph_destroy",
)

if not os.path.exists(_LIB_PATH):
    raise ImportError(f"{_LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(nvcc, sm_100a); there is no CPU fallback")

_lib = ctypes.CDLL(_LIB_PATH)
_P = ctypes.c_void_p
_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int)

_lib.qsim_last_error.restype = ctypes.c_char_p
_lib.qsim_create.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_P)]
_lib.qsim_create_ex.argtypes = [ctypes.POINTER(qsim_config), ctypes.POINTER(_P)]
_lib.qsim_destroy.argtypes = [_P]
_lib.qsim_nccl_unique_id.argtypes = [ctypes.c_void_p]
_lib.qsim_apply_gate.argtypes = [_P, _dp, ctypes.c_int, _ip, ctypes.c_int]
_lib.qsim_apply_swap.argtypes = [_P, ctypes.c_int, ctypes.c_int]
_lib.qsim_apply_circuit.argtypes = [_P, ctypes.POINTER(qsim_gate), ctypes.c_size_t]
_lib.qsim_norm.argtypes = [_P, _dp]
_lib.qsim_probabilities.argtypes = [_P, _dp]
_lib.qsim_expectations.argtypes = [_P, _dp]
_lib.qsim_measure.argtypes = [_P, ctypes.c_int, ctypes.c_uint64, _ip]
_lib.qsim_measure_u.argtypes = [_P, ctypes.c_int, ctypes.c_double, _ip, _dp]
_lib.qsim_project.argtypes = [_P, ctypes.c_int, ctypes.c_int]
_lib.qsim_prepare_shorbox.argtypes = [_P, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64]
_lib.qsim_aux_amplitudes.argtypes = [ctypes.c_int, ctypes.POINTER(qsim_gate), ctypes.c_size_t,
                                     ctypes.POINTER(ctypes.c_uint64), ctypes.c_size_t,
                                     ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
_lib.qsim_set_qubit_map.argtypes = [_P, ctypes.POINTER(ctypes.c_int)]
_lib.qsim_asm_parse.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]
_lib.qsim_asm_info.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int64),
                               ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_double)]
_lib.qsim_asm_get_op.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
_lib.qsim_asm_destroy.argtypes = [ctypes.c_void_p]
_lib.qsim_asm_destroy.restype = None
_lib.qsim_asm_run.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_uint64,
                              ctypes.POINTER(ctypes.c_void_p)]
_lib.qsim_asm_result_get.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64,
                                     ctypes.POINTER(ctypes.c_int64)]
_lib.qsim_asm_result_destroy.argtypes = [ctypes.c_void_p]
_lib.qsim_asm_result_destroy.restype = None
_lib.qsim_aux_num_vars.argtypes = [ctypes.c_int, ctypes.POINTER(qsim_gate), ctypes.c_size_t,
                                   ctypes.POINTER(ctypes.c_int)]
_lib.qsim_sample.argtypes = [_P, ctypes.c_size_t, ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64)]
_lib.qsim_get_amplitudes.argtypes = [_P, ctypes.POINTER(ctypes.c_uint64), ctypes.c_size_t, _dp]
_lib.qsim_get_state.argtypes = [_P, _dp]
_lib.qsim_set_state.argtypes = [_P, _dp]
_lib.qsim_get_codes.argtypes = [_P, ctypes.POINTER(ctypes.c_int8), _dp, _dp]
_lib.qsim_set_codes.argtypes = [_P, ctypes.POINTER(ctypes.c_int8), ctypes.c_double, ctypes.c_double]
_lib.qsim_sync.argtypes = [_P]
_lib.qsim_overlap.argtypes = [_P, _P, _dp]
_lib.qsim_magnitude_range.argtypes = [_P, _dp, _dp]
_lib.qsim_apply_circuit_persistent.argtypes = [_P, ctypes.POINTER(qsim_gate), ctypes.c_size_t]
_lib.qsim_get_bounds.argtypes = [_P, _dp, _dp]
_lib.qsim_apply_matrix.argtypes = [_P, _dp, _ip, ctypes.c_int]
_lib.qsim_jit_sync.argtypes = []
_lib.qsim_jit_shutdown.argtypes = []
# stop the fused-pass compile threads before the C exit handlers run (qsim.h)
atexit.register(_lib.qsim_jit_shutdown)
_lib.qsim_graph_begin.argtypes = [_P]
_lib.qsim_graph_end.argtypes = [_P, ctypes.POINTER(_P)]
_lib.qsim_graph_launch.argtypes = [_P, _P]
_lib.qsim_graph_destroy.argtypes = [_P]
_lib.qsim_stream.argtypes = [_P, ctypes.c_int]
_lib.qsim_stream.restype = ctypes.c_void_p
_lib.qsim_get_stats.argtypes = [_P, ctypes.POINTER(qsim_stats)]
_lib.qsim_reset_stats.argtypes = [_P]
_lib.qsim_get_qubit_map.argtypes = [_P, _ip]
_lib.qsim_reset.argtypes = [_P]
_lib.qsim_reset_basis.argtypes = [_P, ctypes.c_uint64]
_lib.qsim_profile.argtypes = [_P, ctypes.c_int]
_lib.qsim_profile_read.argtypes = [_P, ctypes.POINTER(qsim_kernel_profile), ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
_lib.qsim_plan_create.argtypes = [ctypes.c_int, ctypes.c_int, _ip, ctypes.POINTER(qsim_gate), ctypes.c_size_t,
                                  ctypes.POINTER(_P)]
_lib.qsim_plan_num_ops.argtypes = [_P]
_lib.qsim_plan_num_ops.restype = ctypes.c_int64
_lib.qsim_plan_get_op.argtypes = [_P, ctypes.c_int64, ctypes.POINTER(qsim_plan_op)]
_lib.qsim_plan_final_map.argtypes = [_P, _ip]
_lib.qsim_plan_destroy.argtypes = [_P]
_lib.qsim_plan_destroy.restype = None


def lib():
    return _lib


def lib_path():
    return _LIB_PATH


def _check(rc):
    if rc != QSIM_OK:
        raise QsimError(rc, _lib.qsim_last_error().decode(errors="replace"))
    return rc


def _dptr(a):
    return a.ctypes.data_as(_dp)


def pack_gates(circuit) -> ctypes.Array:
    """Marshal a circuits.Circuit (or a list of (u, target, controls) / ('SWAP', q1, q2))
    into a qsim_gate array."""
    if hasattr(circuit, "kind"):
        n = len(circuit)
        arr = (qsim_gate * max(n, 1))()
        kind, t, t2, nc, ct, u = circuit.kind, circuit.target, circuit.target2, circuit.nctrl, circuit.ctrl, circuit.u
        buf = np.frombuffer(arr, dtype=np.uint8, count=88 * n).reshape(n, 88) if n else None
        if n:
            ints = np.zeros((n, 6), dtype=np.int32)
            ints[:, 0], ints[:, 1], ints[:, 2], ints[:, 3] = kind, t, t2, nc
            ints[:, 4:6] = ct.reshape(n, 2)
            buf[:, :24] = ints.view(np.uint8).reshape(n, 24)
            buf[:, 24:] = np.ascontiguousarray(u.reshape(n, 8)).view(np.uint8).reshape(n, 64)
        return arr, n
    items = list(circuit)
    arr = (qsim_gate * max(len(items), 1))()
    for i, g in enumerate(items):
        if isinstance(g[0], str) and g[0].upper() == "SWAP":
            arr[i].kind, arr[i].target, arr[i].target2 = GATE_SWAP, g[1], g[2]
            continue
        u, t = g[0], g[1]
        ctl = list(g[2]) if len(g) > 2 else []
        u8 = np.ascontiguousarray(np.asarray(u, dtype=np.complex128).reshape(2, 2)).view(np.float64).reshape(8)
        arr[i].kind, arr[i].target, arr[i].target2, arr[i].ncontrols = GATE_U, t, -1, len(ctl)
        for k, c in enumerate(ctl):
            arr[i].controls[k] = c
        for k in range(8):
            arr[i].u[k] = u8[k]
    return arr, len(items)


# ----------------------------------------------------------------------------- C-ABI mirrors


def qsim_nccl_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check(_lib.qsim_nccl_unique_id(buf))
    return bytes(buf)


def qsim_create(n_qubits: int, encoding: int = ENC_FP64, ngpus: int = 1):
    h = _P()
    _check(_lib.qsim_create(n_qubits, encoding, ngpus, ctypes.byref(h)))
    return h


def qsim_create_ex(n_qubits, encoding=ENC_FP64, nshards=1, transport=TRANSPORT_LOCAL, rank=0, device=-1,
                   nccl_id: bytes | None = None, chunk_bytes=0, fuse=1, a_policy=0):
    cfg = qsim_config()
    cfg.n_qubits, cfg.encoding, cfg.nshards, cfg.transport = n_qubits, encoding, nshards, transport
    cfg.rank, cfg.device, cfg.chunk_bytes, cfg.fuse, cfg.a_policy = rank, device, chunk_bytes, fuse, a_policy
    idbuf = None
    if nccl_id is not None:
        idbuf = (ctypes.c_uint8 * 128).from_buffer_copy(nccl_id)
        cfg.nccl_id = ctypes.addressof(idbuf)
    h = _P()
    _check(_lib.qsim_create_ex(ctypes.byref(cfg), ctypes.byref(h)))
    return h


def qsim_destroy(h):
    _lib.qsim_destroy(h)


def qsim_apply_gate(h, u, target, controls=()):
    u8 = np.ascontiguousarray(np.asarray(u, dtype=np.complex128).reshape(2, 2)).view(np.float64).reshape(8)
    c = (ctypes.c_int * 2)(*(list(controls) + [0, 0])[:2])
    _check(_lib.qsim_apply_gate(h, _dptr(u8), target, c, len(controls)))


def qsim_apply_circuit_persistent(h, circuit):
    arr, n = circuit if isinstance(circuit, tuple) else pack_gates(circuit)
    _check(_lib.qsim_apply_circuit_persistent(h, arr, n))


def qsim_apply_swap(h, q1, q2):
    _check(_lib.qsim_apply_swap(h, q1, q2))


def qsim_apply_circuit(h, circuit):
    arr, n = circuit if isinstance(circuit, tuple) else pack_gates(circuit)
    _check(_lib.qsim_apply_circuit(h, arr, n))


def qsim_norm(h) -> float:
    v = ctypes.c_double()
    _check(_lib.qsim_norm(h, ctypes.byref(v)))
    return v.value


def qsim_probabilities(h, n) -> np.ndarray:
    p = np.empty(n, dtype=np.float64)
    _check(_lib.qsim_probabilities(h, _dptr(p)))
    return p


def qsim_expectations(h, n) -> np.ndarray:
    q = np.empty(3 * n, dtype=np.float64)
    _check(_lib.qsim_expectations(h, _dptr(q)))
    return q.reshape(n, 3)


def qsim_measure(h, qubit, seed) -> int:
    o = ctypes.c_int()
    _check(_lib.qsim_measure(h, qubit, seed, ctypes.byref(o)))
    return o.value


def qsim_measure_u(h, qubit, u):
    o, p0 = ctypes.c_int(), ctypes.c_double()
    _check(_lib.qsim_measure_u(h, qubit, float(u), ctypes.byref(o), ctypes.byref(p0)))
    return o.value, p0.value


def qsim_project(h, qubit, value):
    """CLEAR (value=0) / SET (value=1): project and renormalise."""
    _check(_lib.qsim_project(h, qubit, value))


def qsim_aux_num_vars(n_qubits, circuit) -> int:
    """Number of auxiliary variables of the circuit (§4.2; host only)."""
    arr, n = pack_gates(circuit)
    P = ctypes.c_int()
    _check(_lib.qsim_aux_num_vars(n_qubits, arr, n, ctypes.byref(P)))
    return P.value


def qsim_aux_amplitudes(n_qubits, circuit, idx, return_abs_sum=False):
    """<y|psi> at logical indices idx by the auxiliary-variable method
    (§4.2, Eq. appa7) on the current CUDA device; optionally also
    2^-P sum_s |term_s| per amplitude."""
    arr, n = pack_gates(circuit)
    y = np.ascontiguousarray(np.asarray(idx, dtype=np.uint64))
    out = np.empty(2 * len(y))
    ab = np.empty(len(y))
    _check(_lib.qsim_aux_amplitudes(n_qubits, arr, n, y.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), len(y),
                                    out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                    ab.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
    z = out[0::2] + 1j * out[1::2]
    return (z, ab) if return_abs_sum else z


ASM_GATE, ASM_MEASURE_ALL, ASM_EVENTS, ASM_M, ASM_SHORBOX, ASM_CLEAR, ASM_SET, ASM_EXIT = range(8)


class qsim_asm_op(ctypes.Structure):
    _fields_ = [("type", ctypes.c_int32), ("line", ctypes.c_int32), ("args", ctypes.c_int64 * 3),
                ("gate", qsim_gate)]


def asm_parse(text: str) -> dict:
    """Compile an App. B program (host only): N, the BIT
    ASSIGNMENT map, the depolarising-channel parameters and the op list."""
    h = ctypes.c_void_p()
    _check(_lib.qsim_asm_parse(text.encode(), ctypes.byref(h)))
    try:
        n, nops = ctypes.c_int(), ctypes.c_int64()
        _check(_lib.qsim_asm_info(h, ctypes.byref(n), ctypes.byref(nops), None, None))
        perm = (ctypes.c_int * n.value)()
        dep = (ctypes.c_double * 4)()
        _check(_lib.qsim_asm_info(h, None, None, perm, dep))
        ops = []
        op = qsim_asm_op()
        for i in range(nops.value):
            _check(_lib.qsim_asm_get_op(h, i, ctypes.byref(op)))
            g = op.gate
            ops.append(dict(type=op.type, line=op.line, args=list(op.args), target=g.target,
                            controls=[g.controls[k] for k in range(g.ncontrols)],
                            u=np.array(list(g.u)).view(np.complex128).reshape(2, 2)))
        return dict(n=n.value, perm=list(perm), depol=list(dep), ops=ops)
    finally:
        _lib.qsim_asm_destroy(h)


def asm_run(text: str, encoding=ENC_FP64, ngpus=1, seed=0) -> dict:
    """Run an App. B program on a fresh state: BEGIN MEASUREMENT tables
    (K x N x 3: <Qx>, <Qy>, <Qz>), M outcomes [(qubit, outcome)], events."""
    h = ctypes.c_void_p()
    _check(_lib.qsim_asm_parse(text.encode(), ctypes.byref(h)))
    r = ctypes.c_void_p()
    try:
        n = ctypes.c_int()
        _check(_lib.qsim_asm_info(h, ctypes.byref(n), None, None, None))
        _check(_lib.qsim_asm_run(h, encoding, ngpus, seed, ctypes.byref(r)))
    finally:
        _lib.qsim_asm_destroy(h)
    try:
        out = {}
        for what, dt, key in ((0, np.float64, "tables"), (1, np.int32, "outcomes"), (2, np.uint64, "events")):
            cnt = ctypes.c_int64()
            _check(_lib.qsim_asm_result_get(r, what, None, 0, ctypes.byref(cnt)))
            buf = np.empty(cnt.value, dtype=dt)
            _check(_lib.qsim_asm_result_get(r, what, buf.ctypes.data_as(ctypes.c_void_p), cnt.value,
                                            ctypes.byref(cnt)))
            out[key] = buf
        out["tables"] = out["tables"].reshape(-1, n.value, 3)
        out["outcomes"] = [tuple(x) for x in out["outcomes"].reshape(-1, 2).tolist()]
        return out
    finally:
        _lib.qsim_asm_result_destroy(r)


def qsim_prepare_shorbox(h, nx, G, y):
    """SHORBOX: 2^{-nx/2} sum_x |x>|y^x mod G>, x-register = qubits 0..nx-1."""
    _check(_lib.qsim_prepare_shorbox(h, nx, G, y))


def qsim_sample(h, nsamples, seed) -> np.ndarray:
    """GENERATE EVENTS: logical basis indices drawn from |a|^2."""
    out = np.empty(max(int(nsamples), 1), dtype=np.uint64)
    _check(_lib.qsim_sample(h, int(nsamples), int(seed), out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))))
    return out[:int(nsamples)]


def qsim_get_amplitudes(h, idx) -> np.ndarray:
    idx = np.ascontiguousarray(idx, dtype=np.uint64)
    out = np.empty(idx.size, dtype=np.complex128)
    _check(_lib.qsim_get_amplitudes(h, idx.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), idx.size,
                                    _dptr(out.view(np.float64))))
    return out


def qsim_get_state(h, n) -> np.ndarray:
    out = np.empty(1 << n, dtype=np.complex128)
    _check(_lib.qsim_get_state(h, _dptr(out.view(np.float64))))
    return out


def qsim_set_state(h, amps):
    a = np.ascontiguousarray(amps, dtype=np.complex128)
    _check(_lib.qsim_set_state(h, _dptr(a.view(np.float64))))


def qsim_get_codes(h, n):
    codes = np.empty(2 << n, dtype=np.int8)
    r0, r1 = ctypes.c_double(), ctypes.c_double()
    _check(_lib.qsim_get_codes(h, codes.ctypes.data_as(ctypes.POINTER(ctypes.c_int8)), ctypes.byref(r0),
                               ctypes.byref(r1)))
    return codes, r0.value, r1.value


def qsim_set_codes(h, codes, r0, r1):
    c = np.ascontiguousarray(codes, dtype=np.int8)
    _check(_lib.qsim_set_codes(h, c.ctypes.data_as(ctypes.POINTER(ctypes.c_int8)), float(r0), float(r1)))


def qsim_sync(h):
    _check(_lib.qsim_sync(h))


def qsim_jit_sync():
    """Wait for the queued run-time specialisations of the fused pass (qsim_jit_sync)."""
    _check(_lib.qsim_jit_sync())


def qsim_apply_matrix(h, u, qubits):
    """k-qubit unitary (k = len(qubits) <= 3), qubits[0] the most significant matrix index."""
    k = len(qubits)
    m = np.ascontiguousarray(np.asarray(u, dtype=np.complex128).reshape(1 << k, 1 << k)).view(np.float64).reshape(-1)
    q = (ctypes.c_int * k)(*[int(x) for x in qubits])
    _check(_lib.qsim_apply_matrix(h, m.ctypes.data_as(_dp), q, k))


def qsim_jit_shutdown():
    """Stop the fused-pass compile threads (also registered with atexit)."""
    _check(_lib.qsim_jit_shutdown())


def qsim_overlap(ha, hb) -> complex:
    out = (ctypes.c_double * 2)()
    _check(_lib.qsim_overlap(ha, hb, out))
    return complex(out[0], out[1])


def qsim_magnitude_range(h) -> tuple[float, float]:
    lo, hi = ctypes.c_double(), ctypes.c_double()
    _check(_lib.qsim_magnitude_range(h, ctypes.byref(lo), ctypes.byref(hi)))
    return lo.value, hi.value


def qsim_get_bounds(h) -> tuple[float, float]:
    lo, hi = ctypes.c_double(), ctypes.c_double()
    _check(_lib.qsim_get_bounds(h, ctypes.byref(lo), ctypes.byref(hi)))
    return lo.value, hi.value


def qsim_graph_begin(h):
    _check(_lib.qsim_graph_begin(h))


def qsim_graph_end(h):
    g = _P()
    _check(_lib.qsim_graph_end(h, ctypes.byref(g)))
    return g


def qsim_graph_launch(h, g):
    _check(_lib.qsim_graph_launch(h, g))


def qsim_graph_destroy(g):
    _check(_lib.qsim_graph_destroy(g))


def qsim_stream(h, shard=0) -> int:
    return _lib.qsim_stream(h, shard) or 0


def qsim_get_stats(h) -> dict:
    st = qsim_stats()
    _check(_lib.qsim_get_stats(h, ctypes.byref(st)))
    return {name: getattr(st, name) for name, _ in qsim_stats._fields_}


def qsim_reset_stats(h):
    _check(_lib.qsim_reset_stats(h))


def qsim_reset(h):
    _check(_lib.qsim_reset(h))


def qsim_reset_basis(h, x):
    _check(_lib.qsim_reset_basis(h, int(x)))


def qsim_profile(h, enable=True):
    _check(_lib.qsim_profile(h, 1 if enable else 0))


def qsim_profile_read(h) -> dict:
    """{kernel class name: {"launches", "ms", "bytes"}} since the last read."""
    arr = (qsim_kernel_profile * 8)()
    n = ctypes.c_int()
    _check(_lib.qsim_profile_read(h, arr, 8, ctypes.byref(n)))
    return {KERNEL_NAMES[arr[i].kind]: dict(launches=arr[i].launches, ms=arr[i].ms, bytes=arr[i].bytes,
                                            flops=arr[i].flops)
            for i in range(n.value)}


def qsim_get_qubit_map(h, n) -> list:
    pos = (ctypes.c_int * n)()
    _check(_lib.qsim_get_qubit_map(h, pos))
    return list(pos)


def qsim_plan(n_qubits, nshards, circuit, initial_map=None):
    """Host-only planner (no GPU): returns (ops as dicts, final qubit map)."""
    arr, n = pack_gates(circuit)
    im = None
    if initial_map is not None:
        im = (ctypes.c_int * n_qubits)(*initial_map)
    h = _P()
    _check(_lib.qsim_plan_create(n_qubits, nshards, im, arr, n, ctypes.byref(h)))
    try:
        ops = []
        op = qsim_plan_op()
        for i in range(_lib.qsim_plan_num_ops(h)):
            _check(_lib.qsim_plan_get_op(h, i, ctypes.byref(op)))
            ops.append(dict(type=op.type, g=op.g, l=op.l, cls=op.cls, controls=list(op.controls)[:op.ncontrols],
                            gate_index=op.gate_index))
        pos = (ctypes.c_int * n_qubits)()
        _check(_lib.qsim_plan_final_map(h, pos))
        return ops, list(pos)
    finally:
        _lib.qsim_plan_destroy(h)


class State:
    """Convenience wrapper: one handle, methods named after the C-ABI calls."""

    def __init__(self, n_qubits, encoding=ENC_FP64, ngpus=1, **ex):
        """ngpus > 1 without a transport: that many shards on the current
        device (QSIM_TRANSPORT_LOCAL, loopback); transport=TRANSPORT_DEVICES
        spreads them over devices 0..ngpus-1 (qsim_create's default)."""
        self.n = n_qubits
        self.encoding = encoding
        if ex or ngpus > 1:
            self.h = qsim_create_ex(n_qubits, encoding, ngpus, **ex)
        else:
            self.h = qsim_create(n_qubits, encoding, ngpus)

    def close(self):
        if getattr(self, "h", None):
            qsim_destroy(self.h)
            self.h = None

    __del__ = close

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def apply_gate(self, u, target, controls=()):
        qsim_apply_gate(self.h, u, target, controls)
        return self

    def apply_swap(self, q1, q2):
        qsim_apply_swap(self.h, q1, q2)
        return self

    def apply_circuit(self, circuit):
        qsim_apply_circuit(self.h, circuit)
        return self

    def apply_circuit_persistent(self, circuit):
        """The whole circuit in one cluster kernel (qsim_apply_circuit_persistent)."""
        qsim_apply_circuit_persistent(self.h, circuit)
        return self

    def norm(self):
        return qsim_norm(self.h)

    def probabilities(self):
        return qsim_probabilities(self.h, self.n)

    def expectations(self):
        return qsim_expectations(self.h, self.n)

    def measure(self, qubit, seed):
        return qsim_measure(self.h, qubit, seed)

    def measure_u(self, qubit, u):
        return qsim_measure_u(self.h, qubit, u)

    def prepare_shorbox(self, nx, G, y):
        qsim_prepare_shorbox(self.h, nx, G, y)
        return self

    def sample(self, nsamples, seed):
        return qsim_sample(self.h, nsamples, seed)

    def project(self, qubit, value):
        qsim_project(self.h, qubit, value)
        return self

    def get_amplitudes(self, idx):
        return qsim_get_amplitudes(self.h, idx)

    def get_state(self):
        return qsim_get_state(self.h, self.n)

    def set_state(self, amps):
        qsim_set_state(self.h, amps)
        return self

    def get_codes(self):
        return qsim_get_codes(self.h, self.n)

    def set_codes(self, codes, r0, r1):
        qsim_set_codes(self.h, codes, r0, r1)
        return self

    def sync(self):
        qsim_sync(self.h)

    def stream(self, shard=0):
        """cudaStream_t of the handle (of member `shard` for the multi-device transport)."""
        return qsim_stream(self.h, shard)

    def apply_matrix(self, u, qubits):
        qsim_apply_matrix(self.h, u, qubits)
        return self

    def magnitude_range(self):
        """(min non-zero |a|, max |a|) of an E state (qsim_magnitude_range)."""
        return qsim_magnitude_range(self.h)

    def bounds(self):
        """(r0, r1) of an A state (qsim_get_bounds)."""
        return qsim_get_bounds(self.h)

    def overlap(self, other):
        """<self|other> (qsim_overlap)."""
        return qsim_overlap(self.h, other.h)

    def capture(self, fn):
        """Capture the launches fn(self) makes into a CUDA graph (qsim_graph_*);
        returns a Graph whose launch() replays them on the current state."""
        qsim_graph_begin(self.h)
        try:
            fn(self)
        except BaseException:
            try:
                qsim_graph_destroy(qsim_graph_end(self.h))
            except QsimError:
                pass
            raise
        return Graph(self, qsim_graph_end(self.h))

    def stats(self):
        return qsim_get_stats(self.h)

    def reset_stats(self):
        qsim_reset_stats(self.h)

    def reset(self):
        qsim_reset(self.h)
        return self

    def reset_basis(self, x):
        """|x> (logical index x): the state X on the set bits of x makes from |0...0>."""
        qsim_reset_basis(self.h, x)
        return self

    def profile(self, enable=True):
        qsim_profile(self.h, enable)

    def profile_read(self):
        return qsim_profile_read(self.h)

    def qubit_map(self):
        return qsim_get_qubit_map(self.h, self.n)


class Graph:
    """A captured gate sequence (qsim_graph_*): launch() replays it on the
    owning State's stream with no host planning."""

    def __init__(self, state, g):
        self.state, self.g = state, g

    def launch(self):
        qsim_graph_launch(self.state.h, self.g)

    def close(self):
        if self.g:
            qsim_graph_destroy(self.g)
            self.g = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
