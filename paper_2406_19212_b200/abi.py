"""ctypes mirror of include/vqcs_b200.h and the circuit descriptors that cross it.

The same struct layouts are shared by the product library (``libvqcs_b200.so``,
prefix ``vqb_``) and the test-only checkers under ``oracle/`` (prefixes
``vqcsref_`` / ``vqcsorc_``), which implement the identical C-ABI on the CPU.
"""
from __future__ import annotations

import ctypes as ct
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Iterable, Optional, Sequence

import numpy as np

MAX_POSITIONS = 6
MAX_PARAMS = 5


class GateKind(IntEnum):
    """gates.hpp:38-61 (same numbering)."""
    Generic = 0
    X = 1
    Y = 2
    Z = 3
    H = 4
    S = 5
    T = 6
    SqrtX = 7
    SqrtY = 8
    Swap = 9
    ISwap = 10
    CZ = 11
    Cnot = 12
    Toffoli = 13
    Fredkin = 14
    Rx = 15
    Ry = 16
    Rz = 17
    CRx = 18
    CRy = 19
    CRz = 20
    Fsim = 21


class ChannelKind(IntEnum):
    """gates.hpp:63-68."""
    Generic = 0
    AmplitudeDamping = 1
    PhaseDamping = 2
    Depolarizing = 3


ELEM_GATE = 0
ELEM_CHANNEL = 1


class c128(ct.Structure):
    _fields_ = [("re", ct.c_double), ("im", ct.c_double)]


c128_p = ct.POINTER(c128)


class vqb_op(ct.Structure):
    _fields_ = [
        ("elem", ct.c_int32),
        ("kind", ct.c_int32),
        ("num_positions", ct.c_int32),
        ("positions", ct.c_int32 * MAX_POSITIONS),
        ("num_params", ct.c_int32),
        ("params", ct.c_double * MAX_PARAMS),
        ("is_param", ct.c_int32 * MAX_PARAMS),
        ("matrix", c128_p),
        ("num_kraus", ct.c_int32),
        ("kraus", c128_p),
    ]


class vqb_rev_step(ct.Structure):
    """One reverse step (reverse_sweep_step kernels.hpp:659-697) with explicit
    matrices, for vqb_reverse_sweep."""
    _fields_ = [
        ("num_positions", ct.c_int32),
        ("positions", ct.c_int32 * MAX_POSITIONS),
        ("inv", c128_p),
        ("num_dmats", ct.c_int32),
        ("dmats", c128_p),
        ("grad_index", ct.c_int64),
    ]


class vqb_pauli_term(ct.Structure):
    _fields_ = [
        ("coeff", c128),
        ("num_factors", ct.c_int32),
        ("qubits", ct.POINTER(ct.c_int32)),
        ("labels", ct.c_char_p),
    ]


# ---- error taxonomy: errors.hpp:23-96, status codes 1..11 ----
class VqcsError(RuntimeError):
    """Base class, vqcs::Error."""


class SizeError(VqcsError): pass
class ShapeError(VqcsError): pass
class ValidityError(VqcsError): pass
class DomainError(VqcsError): pass
class IndexError_(VqcsError): pass
class TypeError_(VqcsError): pass
class UnsupportedError(VqcsError): pass
class DegenerateStateError(VqcsError): pass
class NonInvertibleChannelError(VqcsError): pass
class IoError(VqcsError): pass
class UsageError(VqcsError): pass
class CudaError(VqcsError): pass
class NcclError(VqcsError): pass
class InternalError(VqcsError): pass


STATUS_TO_ERROR = {
    1: SizeError, 2: ShapeError, 3: ValidityError, 4: DomainError, 5: IndexError_,
    6: TypeError_, 7: UnsupportedError, 8: DegenerateStateError,
    9: NonInvertibleChannelError, 10: IoError, 11: UsageError, 20: CudaError,
    21: NcclError, 22: InternalError,
}


def as_c128_array(mat: np.ndarray) -> np.ndarray:
    """Column-major flattening of a 2^m x 2^m complex matrix (gates.hpp:18-22)."""
    a = np.asarray(mat, dtype=np.complex128)
    if a.ndim == 2:
        a = a.flatten(order="F")
    return np.ascontiguousarray(a, dtype=np.complex128)


def c128_ptr(arr: Optional[np.ndarray]):
    if arr is None:
        return None
    return arr.ctypes.data_as(c128_p)


# ---- circuit elements (GateOp gates.hpp:106-130, ChannelOp :133-141) ----
@dataclass
class GateOp:
    positions: list
    kind: GateKind = GateKind.Generic
    params: list = field(default_factory=list)
    is_param: list = field(default_factory=list)
    matrix: Optional[np.ndarray] = None  # flattened column-major, or None (built from kind)

    def num_targets(self) -> int:
        return len(self.positions)

    def num_active_params(self) -> int:
        return sum(1 for b in self.is_param if b)


@dataclass
class ChannelOp:
    positions: list
    kind: ChannelKind = ChannelKind.Generic
    param: float = 0.0
    kraus: Optional[list] = None  # list of flattened column-major matrices, or None (named)


def standard_gate(kind: GateKind, positions: Sequence[int]) -> GateOp:
    return GateOp(list(positions), GateKind(kind))


def parametric_gate(kind: GateKind, positions: Sequence[int], params, is_param) -> GateOp:
    if np.isscalar(params):
        params, is_param = [float(params)], [bool(is_param)]
    return GateOp(list(positions), GateKind(kind), [float(p) for p in params],
                  [bool(b) for b in is_param])


def make_gate(positions: Sequence[int], matrix) -> GateOp:
    return GateOp(list(positions), GateKind.Generic, matrix=as_c128_array(matrix))


def standard_channel(kind: ChannelKind, position: int, param: float) -> ChannelOp:
    return ChannelOp([position], ChannelKind(kind), float(param))


def make_channel(positions: Sequence[int], kraus: Iterable) -> ChannelOp:
    return ChannelOp(list(positions), ChannelKind.Generic, 0.0,
                     [as_c128_array(k) for k in kraus])


class Circuit:
    """Flattened element list (circuit.hpp:38-106); nested circuits are
    appended in depth-first order, the reference's traversal order."""

    def __init__(self, elements: Iterable = ()):
        self.elements: list = []
        for e in elements:
            self.push_back(e)
        self._packed = None

    def push_back(self, e) -> None:
        if isinstance(e, Circuit):
            self.elements.extend(e.elements)
        else:
            self.elements.append(e)
        self._packed = None

    def __len__(self) -> int:
        return len(self.elements)

    def has_channels(self) -> bool:
        return any(isinstance(e, ChannelOp) for e in self.elements)

    def num_active_params(self) -> int:
        return sum(e.num_active_params() for e in self.elements if isinstance(e, GateOp))

    def active_parameters(self) -> list:
        """circuit.hpp:149-159."""
        out = []
        for e in self.elements:
            if isinstance(e, GateOp):
                out.extend(p for p, b in zip(e.params, e.is_param) if b)
        return out

    def reset_parameters(self, values: Sequence[float]) -> None:
        """circuit.hpp:163-185 (matrices of named kinds are rebuilt from
        params on the native side, so only params change here)."""
        cur = 0
        for e in self.elements:
            if isinstance(e, GateOp):
                for i, b in enumerate(e.is_param):
                    if b:
                        if cur >= len(values):
                            raise ShapeError("reset_parameters: too few values")
                        e.params[i] = float(values[cur])
                        cur += 1
        if cur != len(values):
            raise ShapeError(f"reset_parameters: expected {cur} values, got {len(values)}")
        self._packed = None

    def pack(self):
        """-> (ctypes array of vqb_op, count); buffers kept alive on self."""
        if self._packed is None:
            self._packed = pack_ops(self.elements)
        return self._packed


class PackedOps:
    def __init__(self, arr, count, keep):
        self.arr = arr
        self.count = count
        self._keep = keep

    @property
    def ptr(self):
        return self.arr


def pack_ops(elements: Sequence) -> PackedOps:
    n = len(elements)
    arr = (vqb_op * max(n, 1))()
    keep = []
    for i, e in enumerate(elements):
        o = arr[i]
        if len(e.positions) > MAX_POSITIONS:
            raise UnsupportedError("more than 6 positions")
        o.num_positions = len(e.positions)
        for k, p in enumerate(e.positions):
            o.positions[k] = int(p)
        if isinstance(e, GateOp):
            o.elem = ELEM_GATE
            o.kind = int(e.kind)
            o.num_params = len(e.params)
            for k, (p, b) in enumerate(zip(e.params, e.is_param)):
                o.params[k] = p
                o.is_param[k] = 1 if b else 0
            if e.matrix is not None:
                m = as_c128_array(e.matrix)
                keep.append(m)
                o.matrix = c128_ptr(m)
        else:
            o.elem = ELEM_CHANNEL
            o.kind = int(e.kind)
            o.num_params = 1
            o.params[0] = e.param
            if e.kraus is not None:
                k = np.ascontiguousarray(np.concatenate([as_c128_array(x) for x in e.kraus]))
                keep.append(k)
                o.kraus = c128_ptr(k)
                o.num_kraus = len(e.kraus)
    return PackedOps(arr, n, keep)


# ---- observables (observables.hpp:38-110) ----
@dataclass
class PauliTerm:
    factors: list  # [(qubit, 'x'|'y'|'z'), ...]
    coeff: complex = 1.0


class PauliOperator:
    def __init__(self, terms: Iterable[PauliTerm] = ()):
        self.terms = list(terms)
        self._packed = None

    def add_term(self, t: PauliTerm) -> None:
        self.terms.append(t)
        self._packed = None

    def __len__(self):
        return len(self.terms)

    def conjugated(self) -> "PauliOperator":
        return PauliOperator([PauliTerm(list(t.factors), complex(t.coeff).conjugate())
                              for t in self.terms])

    def pack(self):
        if self._packed is None:
            arr = (vqb_pauli_term * max(len(self.terms), 1))()
            keep = []
            for i, t in enumerate(self.terms):
                q = (ct.c_int32 * max(len(t.factors), 1))(*[int(f[0]) for f in t.factors])
                lab = ct.c_char_p(bytes("".join(str(f[1]) for f in t.factors), "ascii"))
                keep += [q, lab]
                c = complex(t.coeff)
                arr[i].coeff.re, arr[i].coeff.im = c.real, c.imag
                arr[i].num_factors = len(t.factors)
                arr[i].qubits = ct.cast(q, ct.POINTER(ct.c_int32))
                arr[i].labels = lab
            self._packed = (arr, len(self.terms), keep)
        return self._packed


def sum_z(n: int) -> PauliOperator:
    """H = sum_i Z_i (configs 0 and 3)."""
    return PauliOperator([PauliTerm([(q, "z")], 1.0) for q in range(1, n + 1)])


def heisenberg_1d(length: int, hz: float = 1.0, J: float = 1.0) -> PauliOperator:
    """observables.hpp:114-128."""
    if length < 1:
        raise DomainError("heisenberg_1d: length must be >= 1")
    op = PauliOperator()
    for i in range(1, length + 1):
        op.add_term(PauliTerm([(i, "z")], hz))
    for i in range(1, length):
        for l in "xyz":
            op.add_term(PauliTerm([(i, l), (i + 1, l)], J))
    return op


# ---- binding helper shared by product and oracle libraries ----
class vqb_bench_record(ct.Structure):
    _fields_ = [("task", ct.c_char_p), ("num_qubits", ct.c_int32), ("depth", ct.c_int32),
                ("threads", ct.c_int32), ("seconds", ct.POINTER(ct.c_double)), ("num_seconds", ct.c_int64),
                ("speedup", ct.c_double), ("num_info", ct.c_int64),
                ("info_keys", ct.POINTER(ct.c_char_p)), ("info_values", ct.POINTER(ct.c_char_p))]


def pack_bench_records(records):
    """[{task, n, depth, threads, seconds: [...], speedup?, params: {k: v}}]
    -> (ctypes array, keep-alive list)."""
    keep = []
    arr = (vqb_bench_record * max(len(records), 1))()
    for i, r in enumerate(records):
        secs = (ct.c_double * max(len(r["seconds"]), 1))(*r["seconds"])
        items = sorted((str(k), str(v)) for k, v in r.get("params", {}).items())
        kb = [k.encode() for k, _ in items]  # the arrays point into these: keep them alive
        vb = [v.encode() for _, v in items]
        keys = (ct.c_char_p * max(len(items), 1))(*kb)
        vals = (ct.c_char_p * max(len(items), 1))(*vb)
        task = r["task"].encode()
        keep += [secs, keys, vals, task, kb, vb]
        arr[i] = vqb_bench_record(task, int(r["n"]), int(r["depth"]), int(r["threads"]), secs,
                                  len(r["seconds"]), float(r.get("speedup", 0.0)), len(items), keys, vals)
    return arr, keep


def bind_abi(lib: ct.CDLL, prefix: str) -> None:
    """Declare argtypes/restype for every ABI function the library exports."""
    vp = ct.c_void_p
    i32, i64, u64 = ct.c_int32, ct.c_int64, ct.c_uint64
    op_p = ct.POINTER(vqb_op)
    term_p = ct.POINTER(vqb_pauli_term)
    dp = ct.POINTER(ct.c_double)
    sig = {
        "last_error": (ct.c_char_p, []),
        "state_create": (ct.c_int, [i32, i32, ct.POINTER(vp)]),
        "state_destroy": (ct.c_int, [vp]),
        "state_info": (ct.c_int, [vp, ct.POINTER(i32), ct.POINTER(i32), ct.POINTER(u64)]),
        "state_upload": (ct.c_int, [vp, c128_p, u64]),
        "state_upload_async": (ct.c_int, [vp, c128_p, u64]),
        "state_download": (ct.c_int, [vp, c128_p, u64]),
        "state_copy": (ct.c_int, [vp, vp]),
        "state_download_range": (ct.c_int, [vp, u64, u64, c128_p]),
        "apply_gate": (ct.c_int, [vp, op_p]),
        "apply_channel": (ct.c_int, [vp, op_p]),
        "apply_matrix": (ct.c_int, [vp, ct.POINTER(i32), i32, c128_p]),
        "apply_circuit": (ct.c_int, [vp, op_p, i64]),
        "norm": (ct.c_int, [vp, dp]),
        "trace": (ct.c_int, [vp, c128_p]),
        "expectation": (ct.c_int, [vp, term_p, i64, c128_p]),
        "apply_operator": (ct.c_int, [vp, vp, term_p, i64]),
        "bilinear_form": (ct.c_int, [vp, vp, ct.POINTER(i32), i32, c128_p, c128_p]),
        "reverse_step": (ct.c_int, [vp, vp, ct.POINTER(i32), i32, c128_p, c128_p, i32, c128_p]),
        "loss_pure": (ct.c_int, [op_p, i64, term_p, i64, vp, dp]),
        "gradient_pure": (ct.c_int, [op_p, i64, term_p, i64, vp, dp, dp, i64,
                                     ct.POINTER(i64), dp]),
        "loss_mixed": (ct.c_int, [op_p, i64, term_p, i64, vp, dp]),
        "gradient_mixed": (ct.c_int, [op_p, i64, term_p, i64, vp, dp, dp, i64,
                                      ct.POINTER(i64), dp]),
        "gate_matrix": (ct.c_int, [op_p, c128_p]),
        "gate_derivative": (ct.c_int, [op_p, i32, c128_p]),
        "gate_inverse": (ct.c_int, [op_p, c128_p]),
        "channel_superop": (ct.c_int, [op_p, c128_p]),
        "channel_inverse": (ct.c_int, [op_p, c128_p, dp, ct.POINTER(i32)]),
        "bench_report": (ct.c_int, [ct.POINTER(vqb_bench_record), i64, i32, ct.c_char_p, i64, ct.POINTER(i64)]),
        "measure": (ct.c_int, [vp, i32, ct.c_double, ct.POINTER(i32), dp]),
        "measure_probability": (ct.c_int, [vp, i32, dp]),
        "collapse": (ct.c_int, [vp, i32, i32, ct.c_double]),
        "state_save": (ct.c_int, [vp, ct.c_char_p]),
        "state_load": (ct.c_int, [ct.c_char_p, ct.POINTER(vp), ct.POINTER(i32)]),
        "fuse_gates": (ct.c_int, [op_p, i64, i64, op_p, i64, c128_p, ct.POINTER(i64),
                                  ct.POINTER(i64)]),
        "reverse_sweep": (ct.c_int, [vp, vp, ct.POINTER(vqb_rev_step), i64, ct.c_double, dp, i64]),
        # product-only
        "state_wrap": (ct.c_int, [vp, i32, i32, u64, i32, ct.POINTER(vp)]),
        "sharded_create": (ct.c_int, [i32, i32, ct.POINTER(i32), ct.POINTER(vp)]),
        "sharded_destroy": (ct.c_int, [vp]),
        "sharded_set_zero": (ct.c_int, [vp]),
        "sharded_apply_circuit": (ct.c_int, [vp, op_p, i64]),
        "sharded_norm": (ct.c_int, [vp, dp]),
        "sharded_expectation": (ct.c_int, [vp, term_p, i64, c128_p]),
        "sharded_download": (ct.c_int, [vp, c128_p, u64]),
        "sharded_upload": (ct.c_int, [vp, c128_p, u64]),
        "sharded_save": (ct.c_int, [vp, ct.c_char_p]),
        "sharded_gradient_pure": (ct.c_int, [vp, op_p, i64, term_p, i64, dp, dp, i64, ct.POINTER(i64)]),
        "sharded_load": (ct.c_int, [vp, ct.c_char_p, ct.POINTER(i32)]),
        "sharded_stats": (ct.c_int, [vp, ct.POINTER(i64), ct.POINTER(i64), ct.POINTER(u64), ct.POINTER(i32)]),
        "alloc_stats": (ct.c_int, [ct.POINTER(i64), ct.POINTER(i64), ct.POINTER(u64), ct.POINTER(u64)]),
        "reset_alloc_peak": (ct.c_int, []),
        "release_caches": (ct.c_int, []),
        "state_device_ptr": (ct.c_int, [vp, ct.POINTER(vp)]),
        "state_set_zero": (ct.c_int, [vp]),
        "apply_circuit_unfused": (ct.c_int, [vp, op_p, i64]),
        "apply_circuit_copy_batch": (ct.c_int, [i32, i32, op_p, i64, ct.POINTER(c128_p), ct.POINTER(c128_p), i64]),
        "build_info": (ct.c_char_p, []),
        "kernel_launch_count": (i64, []),
        "flop_count": (ct.c_double, []),
        "debug_jit_source": (ct.c_int, [ct.c_int32, ct.c_void_p, ct.c_size_t, ct.c_int32, ct.c_char_p,
                                        ct.c_size_t, ct.POINTER(ct.c_double)]),
        "profile_begin": (ct.c_int, []),
        "profile_end": (ct.c_int, [ct.c_char_p, i64]),
        "state_stream": (ct.c_int, [vp, ct.POINTER(vp)]),
        "plan_blocks": (ct.c_int, [op_p, i64, i32, i32, i32, i32, i64, ct.POINTER(i64),
                                   ct.POINTER(i64), ct.POINTER(i32), ct.POINTER(i32), c128_p]),
        # oracle-only
        "apply_gate_naive": (ct.c_int, [vp, op_p]),
        "uniform_unit": (ct.c_int, [u64, u64, dp]),
        "measure_seeded": (ct.c_int, [vp, i32, u64, u64, ct.POINTER(i32), dp]),
        "set_num_threads": (None, [ct.c_int]),
        "get_num_threads": (ct.c_int, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, prefix + name, None)
        if fn is None:
            continue
        fn.restype = res
        fn.argtypes = args


ABI_FUNCTIONS = [
    "last_error", "build_info", "kernel_launch_count", "flop_count", "debug_jit_source", "profile_begin", "profile_end",
    "state_stream", "alloc_stats", "reset_alloc_peak", "release_caches", "state_create", "state_wrap",
    "state_destroy", "state_info", "state_device_ptr", "state_set_zero", "state_upload",
    "state_download", "state_download_range", "state_copy", "apply_gate", "apply_channel", "apply_matrix",
    "apply_circuit", "apply_circuit_unfused", "apply_circuit_copy_batch", "norm", "trace", "expectation",
    "apply_operator", "bilinear_form", "reverse_step", "loss_pure", "gradient_pure",
    "loss_mixed", "gradient_mixed", "gate_matrix", "gate_derivative", "gate_inverse",
    "channel_superop", "plan_blocks", "measure", "measure_probability", "collapse",
    "state_save", "state_load", "fuse_gates", "reverse_sweep",
]
