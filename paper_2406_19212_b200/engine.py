"""Python binding over one implementation of the include/vqcs_b200.h C-ABI.

`Engine(lib, prefix)` wraps a loaded library; the product binds
``libvqcs_b200.so`` (prefix ``vqb_``), and the test-only ``oracle`` package
binds the CPU checkers with the same class, so parity tests call both sides
through identical Python code. Method names follow the reference API
(apply_circuit, expectation, gradient_pure, ... in namespace vqcs).
"""
from __future__ import annotations

import ctypes as ct
from typing import Optional, Sequence

import numpy as np

from . import abi
from .abi import Circuit, PauliOperator, c128, c128_p, pack_ops


class State:
    """A state handle: PureState<double> (mixed=False) or MixedState<double>."""

    def __init__(self, engine: "Engine", handle: ct.c_void_p, n: int, mixed: bool):
        self.engine = engine
        self.handle = handle
        self.n = n
        self.mixed = mixed

    @property
    def num_qubits(self) -> int:
        return self.n

    @property
    def size(self) -> int:
        return 1 << (2 * self.n if self.mixed else self.n)

    def amplitudes(self) -> np.ndarray:
        return self.engine.download(self)

    def free(self) -> None:
        if self.handle:
            self.engine._fn("state_destroy")(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class ShardedHandle:
    """vqb_sharded: one process, P = 2^g devices (include/vqcs_b200.h)."""

    def __init__(self, engine: "Engine", n: int, devices):
        self.engine = engine
        self.n = n
        self.devices = list(devices)
        h = ct.c_void_p()
        dv = (ct.c_int32 * len(self.devices))(*self.devices)
        engine.check(engine._fn("sharded_create")(n, len(self.devices), dv, ct.byref(h)))
        self.handle = h

    def _f(self, name):
        return self.engine._fn("sharded_" + name)

    def set_zero(self) -> None:
        self.engine.check(self._f("set_zero")(self.handle))

    def apply_circuit(self, c: Circuit) -> None:
        p = c.pack() if isinstance(c, Circuit) else pack_ops(c)
        self.engine.check(self._f("apply_circuit")(self.handle, p.arr, p.count))

    def norm(self) -> float:
        v = ct.c_double()
        self.engine.check(self._f("norm")(self.handle, ct.byref(v)))
        return v.value

    def expectation(self, op: PauliOperator) -> complex:
        arr, nt, _k = op.pack()
        v = c128()
        self.engine.check(self._f("expectation")(self.handle, arr, nt, ct.byref(v)))
        return complex(v.re, v.im)

    def download(self) -> np.ndarray:
        out = np.empty(1 << self.n, dtype=np.complex128)
        self.engine.check(self._f("download")(self.handle, out.ctypes.data_as(c128_p), ct.c_uint64(out.size)))
        return out

    def upload(self, amps: np.ndarray) -> None:
        amps = np.ascontiguousarray(amps, dtype=np.complex128)
        self.engine.check(self._f("upload")(self.handle, amps.ctypes.data_as(c128_p), ct.c_uint64(amps.size)))

    def save(self, path: str) -> None:
        self.engine.check(self._f("save")(self.handle, path.encode()))

    def gradient_pure(self, op: PauliOperator, c: Circuit):
        """gradient_pure with this state as s0 (left as the reverse-swept Phi)
        -> (loss, grads)."""
        p = c.pack() if isinstance(c, Circuit) else pack_ops(c)
        arr, nt, _k = op.pack()
        cap = max(1, c.num_active_params() if isinstance(c, Circuit) else 4096)
        grads = np.zeros(cap, dtype=np.float64)
        loss, ng = ct.c_double(), ct.c_int64()
        self.engine.check(self._f("gradient_pure")(self.handle, p.arr, p.count, arr, nt, ct.byref(loss),
                                                   grads.ctypes.data_as(ct.POINTER(ct.c_double)), cap,
                                                   ct.byref(ng)))
        return loss.value, grads[:ng.value]

    def load(self, path: str) -> int:
        p = ct.c_int32()
        self.engine.check(self._f("load")(self.handle, path.encode(), ct.byref(p)))
        return p.value

    def stats(self) -> dict:
        r, b = ct.c_int64(), ct.c_int64()
        m = ct.c_uint64()
        lp = (ct.c_int32 * self.n)()
        self.engine.check(self._f("stats")(self.handle, ct.byref(r), ct.byref(b), ct.byref(m), lp))
        return {"rounds": r.value, "swapped_bits": b.value, "bytes_moved": m.value, "log2phys": list(lp)}

    def free(self) -> None:
        if self.handle:
            self.engine._fn("sharded_destroy")(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Engine:
    def __init__(self, lib: ct.CDLL, prefix: str, name: str):
        self.lib = lib
        self.prefix = prefix
        self.name = name
        abi.bind_abi(lib, prefix)

    # ---- plumbing ----
    def _fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def has(self, name: str) -> bool:
        return hasattr(self.lib, self.prefix + name)

    def check(self, rc: int) -> None:
        if rc != 0:
            msg = self._fn("last_error")()
            msg = msg.decode() if msg else ""
            raise abi.STATUS_TO_ERROR.get(rc, abi.InternalError)(f"[{self.name}] {msg}")

    # ---- instrumentation (product library only) ----
    def launch_count(self) -> int:
        return int(self._fn("kernel_launch_count")())

    def flop_count(self) -> float:
        return float(self._fn("flop_count")())

    def profile_begin(self) -> None:
        self.check(self._fn("profile_begin")())

    def profile_end(self, launches: Optional[list] = None) -> dict:
        """-> {kernel name: (launches, total_ms)} for the window; annotated
        launches (stage kernels: name, ms, FP64 flops, HBM bytes) are appended
        to `launches` when given."""
        buf = ct.create_string_buffer(1 << 20)
        self.check(self._fn("profile_end")(buf, len(buf)))
        out = {}
        for line in buf.value.decode().splitlines():
            if line.startswith("#L "):
                if launches is not None:
                    _, name, ms, fl, by = line.split()
                    launches.append((name, float(ms), float(fl), float(by)))
                continue
            name, cnt, ms = line.split()
            out[name] = (int(cnt), float(ms))
        return out

    def sharded(self, n: int, devices) -> ShardedHandle:
        """A pure n-qubit state sharded over `devices` (vqb_sharded_create)."""
        return ShardedHandle(self, n, devices)

    def alloc_stats(self) -> dict:
        """state_alloc_stats (state.hpp:154-161) plus device bytes."""
        a, b = ct.c_int64(), ct.c_int64()
        c, d = ct.c_uint64(), ct.c_uint64()
        self.check(self._fn("alloc_stats")(ct.byref(a), ct.byref(b), ct.byref(c), ct.byref(d)))
        return {"live": a.value, "peak": b.value, "live_bytes": c.value, "peak_bytes": d.value}

    def reset_alloc_peak(self) -> None:
        self.check(self._fn("reset_alloc_peak")())

    def release_caches(self) -> None:
        self.check(self._fn("release_caches")())

    def stream_of(self, s: "State") -> int:
        v = ct.c_void_p()
        self.check(self._fn("state_stream")(s.handle, ct.byref(v)))
        return v.value or 0

    # ---- states ----
    def create(self, n: int, mixed: bool = False) -> State:
        h = ct.c_void_p()
        self.check(self._fn("state_create")(n, 1 if mixed else 0, ct.byref(h)))
        return State(self, h, n, mixed)

    def pure_state(self, n: int) -> State:
        return self.create(n, False)

    def mixed_state(self, n: int) -> State:
        return self.create(n, True)

    def from_amplitudes(self, amps: np.ndarray, mixed: bool = False) -> State:
        amps = np.ascontiguousarray(amps, dtype=np.complex128)
        nb = int(amps.size).bit_length() - 1
        n = nb // 2 if mixed else nb
        s = self.create(n, mixed)
        self.upload(s, amps)
        return s

    def upload(self, s: State, amps: np.ndarray) -> None:
        amps = np.ascontiguousarray(amps, dtype=np.complex128)
        self.check(self._fn("state_upload")(s.handle, amps.ctypes.data_as(c128_p),
                                            ct.c_uint64(amps.size)))

    def upload_async(self, s: State, pinned_ptr: int, count: int) -> None:
        """vqb_state_upload_async: `pinned_ptr` addresses page-locked host
        memory that stays unchanged until the next result-returning call on `s`
        (product only; the CPU checkers have no such entry point)."""
        self.check(self._fn("state_upload_async")(s.handle, ct.cast(ct.c_void_p(pinned_ptr), c128_p),
                                                  ct.c_uint64(count)))

    def download(self, s: State, out: Optional[np.ndarray] = None) -> np.ndarray:
        if out is None:
            out = np.empty(s.size, dtype=np.complex128)
        self.check(self._fn("state_download")(s.handle, out.ctypes.data_as(c128_p),
                                              ct.c_uint64(out.size)))
        return out

    def set_zero(self, s: State) -> None:
        """Back to |0...0> (the reference harness's std::fill reset,
        src/bench.cpp:138-141)."""
        self.check(self._fn("state_set_zero")(s.handle))

    def download_range(self, s: State, offset: int, count: int,
                       out: Optional[np.ndarray] = None) -> np.ndarray:
        """Amplitudes [offset, offset + count) (canonical order)."""
        if out is None:
            out = np.empty(count, dtype=np.complex128)
        self.check(self._fn("state_download_range")(s.handle, ct.c_uint64(offset), ct.c_uint64(count),
                                                    out.ctypes.data_as(c128_p)))
        return out

    def copy(self, s: State) -> State:
        d = self.create(s.n, s.mixed)
        self.check(self._fn("state_copy")(d.handle, s.handle))
        return d

    # ---- application ----
    def apply_gate(self, s: State, g) -> None:
        p = pack_ops([g])
        self.check(self._fn("apply_gate")(s.handle, p.arr))

    def apply_gate_naive(self, s: State, g) -> None:
        p = pack_ops([g])
        self.check(self._fn("apply_gate_naive")(s.handle, p.arr))

    def apply_channel(self, s: State, c) -> None:
        p = pack_ops([c])
        self.check(self._fn("apply_channel")(s.handle, p.arr))

    def apply_matrix(self, s: State, positions: Sequence[int], matrix) -> None:
        m = abi.as_c128_array(matrix)
        pos = (ct.c_int32 * len(positions))(*positions)
        self.check(self._fn("apply_matrix")(s.handle, pos, len(positions), abi.c128_ptr(m)))

    def apply_circuit(self, c: Circuit, s: State, fused: bool = True) -> None:
        p = c.pack() if isinstance(c, Circuit) else pack_ops(c)
        name = "apply_circuit" if (fused or not self.has("apply_circuit_unfused")) \
            else "apply_circuit_unfused"
        self.check(self._fn(name)(s.handle, p.arr, p.count))

    def apply_circuit_copy_batch(self, c: Circuit, n: int, inputs, outputs, mixed: bool = False) -> None:
        """apply_circuit_copy (circuit.hpp:132-146) over host states:
        outputs[j] <- c(inputs[j]); inputs/outputs are complex128 numpy arrays
        or raw host addresses (ints, e.g. pinned torch tensors' data_ptr())."""
        p = c.pack() if isinstance(c, Circuit) else pack_ops(c)
        keep = []

        def ptr(x, writable):
            if isinstance(x, int):
                return ct.cast(ct.c_void_p(x), c128_p)
            a = np.asarray(x)
            if a.dtype != np.complex128 or not a.flags.c_contiguous or (writable and not a.flags.writeable):
                raise ValueError("apply_circuit_copy_batch: complex128 C-contiguous arrays required")
            keep.append(a)
            return a.ctypes.data_as(c128_p)
        nb = len(inputs)
        if len(outputs) != nb:
            raise ValueError("apply_circuit_copy_batch: inputs and outputs differ in length")
        ins = (c128_p * max(nb, 1))(*[ptr(x, False) for x in inputs])
        outs = (c128_p * max(nb, 1))(*[ptr(x, True) for x in outputs])
        self.check(self._fn("apply_circuit_copy_batch")(n, 1 if mixed else 0, p.arr, p.count, ins, outs, nb))

    # ---- reductions ----
    def norm(self, s: State) -> float:
        v = ct.c_double()
        self.check(self._fn("norm")(s.handle, ct.byref(v)))
        return v.value

    def trace(self, s: State) -> complex:
        v = c128()
        self.check(self._fn("trace")(s.handle, ct.byref(v)))
        return complex(v.re, v.im)

    def expectation(self, op: PauliOperator, s: State) -> complex:
        arr, nt, _k = op.pack()
        v = c128()
        self.check(self._fn("expectation")(s.handle, arr, nt, ct.byref(v)))
        return complex(v.re, v.im)

    def apply_operator(self, op: PauliOperator, s: State) -> State:
        arr, nt, _k = op.pack()
        out = self.create(s.n, s.mixed)
        self.check(self._fn("apply_operator")(s.handle, out.handle, arr, nt))
        return out

    def bilinear_form(self, bra: State, ket: State, positions, local) -> complex:
        m = abi.as_c128_array(local)
        pos = (ct.c_int32 * len(positions))(*positions)
        v = c128()
        self.check(self._fn("bilinear_form")(bra.handle, ket.handle, pos, len(positions),
                                             abi.c128_ptr(m), ct.byref(v)))
        return complex(v.re, v.im)

    def reverse_step(self, phi: State, psi: State, positions, inv, dmats) -> list:
        iv = abi.as_c128_array(inv)
        dm = np.ascontiguousarray(np.concatenate([abi.as_c128_array(d) for d in dmats]))
        pos = (ct.c_int32 * len(positions))(*positions)
        out = (c128 * max(len(dmats), 1))()
        self.check(self._fn("reverse_step")(phi.handle, psi.handle, pos, len(positions),
                                            abi.c128_ptr(iv), abi.c128_ptr(dm), len(dmats),
                                            out))
        return [complex(out[i].re, out[i].im) for i in range(len(dmats))]

    def reverse_sweep(self, phi: State, psi: State, steps, scale: float, grads: np.ndarray) -> None:
        """Batched reverse steps; steps = [(positions, inv, [dmats], grad_index)],
        grads (float64, C-contiguous) accumulates scale * Re<psi|D|phi>."""
        keep = []
        arr = (abi.vqb_rev_step * max(len(steps), 1))()
        for i, (pos, inv, dmats, gidx) in enumerate(steps):
            st = arr[i]
            st.num_positions = len(pos)
            for k, q in enumerate(pos):
                st.positions[k] = int(q)
            iv = abi.as_c128_array(inv)
            keep.append(iv)
            st.inv = abi.c128_ptr(iv)
            st.num_dmats = len(dmats)
            if dmats:
                dm = np.ascontiguousarray(np.concatenate([abi.as_c128_array(d) for d in dmats]))
                keep.append(dm)
                st.dmats = abi.c128_ptr(dm)
            st.grad_index = int(gidx)
        assert grads.dtype == np.float64 and grads.flags.c_contiguous
        self.check(self._fn("reverse_sweep")(phi.handle, psi.handle, arr, len(steps), float(scale),
                                             grads.ctypes.data_as(ct.POINTER(ct.c_double)),
                                             grads.size))

    # ---- losses / gradients ----
    def loss_pure(self, op: PauliOperator, c: Circuit, s0: State) -> float:
        p = c.pack()
        arr, nt, _k = op.pack()
        v = ct.c_double()
        self.check(self._fn("loss_pure")(p.arr, p.count, arr, nt, s0.handle, ct.byref(v)))
        return v.value

    def loss_mixed(self, op: PauliOperator, c: Circuit, dm0: State) -> float:
        p = c.pack()
        arr, nt, _k = op.pack()
        v = ct.c_double()
        self.check(self._fn("loss_mixed")(p.arr, p.count, arr, nt, dm0.handle, ct.byref(v)))
        return v.value

    def _gradient(self, fn, op, c, s0, with_residual):
        p = c.pack()
        arr, nt, _k = op.pack()
        cap = max(c.num_active_params(), 1)
        grads = np.zeros(cap, dtype=np.float64)
        loss = ct.c_double()
        ng = ct.c_int64()
        res = ct.c_double()
        self.check(self._fn(fn)(p.arr, p.count, arr, nt, s0.handle, ct.byref(loss),
                                grads.ctypes.data_as(ct.POINTER(ct.c_double)), cap,
                                ct.byref(ng), ct.byref(res) if with_residual else None))
        g = grads[: ng.value].copy()
        if with_residual:
            return loss.value, g, res.value
        return loss.value, g

    def gradient_pure(self, op, c, s0, with_residual=False):
        return self._gradient("gradient_pure", op, c, s0, with_residual)

    def gradient_mixed(self, op, c, dm0, with_residual=False):
        return self._gradient("gradient_mixed", op, c, dm0, with_residual)

    # ---- measurement (circuit.hpp:303-375) ----
    def measure(self, s: State, qubit: int, uniform: float):
        """Collapse `qubit` given the reference's uniform draw -> (outcome, p)."""
        o, p = ct.c_int32(), ct.c_double()
        self.check(self._fn("measure")(s.handle, qubit, uniform, ct.byref(o), ct.byref(p)))
        return o.value, p.value

    def measure_probability(self, s: State, qubit: int) -> float:
        p = ct.c_double()
        self.check(self._fn("measure_probability")(s.handle, qubit, ct.byref(p)))
        return p.value

    def collapse(self, s: State, qubit: int, outcome: int, probability: float) -> None:
        self.check(self._fn("collapse")(s.handle, qubit, outcome, probability))

    # ---- state dumps (io.hpp) ----
    def save_state(self, s: State, path: str) -> None:
        self.check(self._fn("state_save")(s.handle, str(path).encode()))

    def load_state(self, path: str):
        """-> (State, precision tag)."""
        h = ct.c_void_p()
        prec = ct.c_int32()
        self.check(self._fn("state_load")(str(path).encode(), ct.byref(h), ct.byref(prec)))
        n = ct.c_int32()
        self.check(self._fn("state_info")(h, ct.byref(n), None, None))
        return State(self, h, n.value, False), prec.value

    # ---- fuse_gates (circuit.hpp:199-276) ----
    def fuse_gates(self, c) -> Circuit:
        p = c.pack() if isinstance(c, Circuit) else pack_ops(c)
        nout, nent = ct.c_int64(), ct.c_int64()
        fn = self._fn("fuse_gates")
        self.check(fn(p.arr, p.count, 0, None, 0, None, ct.byref(nout), ct.byref(nent)))
        ops = (abi.vqb_op * max(nout.value, 1))()
        mats = np.zeros(max(nent.value, 1), dtype=np.complex128)
        self.check(fn(p.arr, p.count, max(nout.value, 1), ops, max(nent.value, 1),
                      mats.ctypes.data_as(c128_p), ct.byref(nout), ct.byref(nent)))
        out = Circuit()
        off = 0
        for i in range(nout.value):
            m = ops[i].num_positions
            d = 1 << m
            out.push_back(abi.make_gate([ops[i].positions[k] for k in range(m)],
                                        mats[off: off + d * d].copy()))
            off += d * d
        return out

    # ---- host-only planning (product library) ----
    def plan_blocks(self, c: Circuit, n: int, mixed: bool = False, tile_bits: int = 12,
                    max_support: int = 2):
        """-> (blocks [(positions, column-major matrix)], num_stages) exactly as
        the fused executor would run them; no device work."""
        p = c.pack() if isinstance(c, Circuit) else pack_ops(c)
        nb, ns = ct.c_int64(), ct.c_int64()
        fn = self._fn("plan_blocks")
        self.check(fn(p.arr, p.count, n, int(mixed), tile_bits, max_support, 0, ct.byref(nb),
                      ct.byref(ns), None, None, None))
        cap = nb.value
        npos = np.zeros(max(cap, 1), dtype=np.int32)
        pos = np.zeros(6 * max(cap, 1), dtype=np.int32)
        mats = np.zeros(256 * max(cap, 1), dtype=np.complex128)
        self.check(fn(p.arr, p.count, n, int(mixed), tile_bits, max_support, cap, ct.byref(nb),
                      ct.byref(ns), npos.ctypes.data_as(ct.POINTER(ct.c_int32)),
                      pos.ctypes.data_as(ct.POINTER(ct.c_int32)), mats.ctypes.data_as(c128_p)))
        blocks = []
        for b in range(nb.value):
            m = int(npos[b])
            d = 1 << m
            blocks.append((list(pos[6 * b: 6 * b + m]), mats[256 * b: 256 * b + d * d].copy()))
        return blocks, ns.value

    # ---- gate algebra ----
    def _mat_call(self, fn, op, dim, *extra):
        out = np.zeros(dim * dim, dtype=np.complex128)
        p = pack_ops([op])
        self.check(self._fn(fn)(p.arr, *extra, out.ctypes.data_as(c128_p)))
        return out

    def gate_matrix(self, g) -> np.ndarray:
        return self._mat_call("gate_matrix", g, 1 << len(g.positions))

    def gate_derivative(self, g, p: int) -> np.ndarray:
        return self._mat_call("gate_derivative", g, 1 << len(g.positions), p)

    def gate_inverse(self, g) -> np.ndarray:
        return self._mat_call("gate_inverse", g, 1 << len(g.positions))

    def channel_superop(self, c) -> np.ndarray:
        return self._mat_call("channel_superop", c, 1 << (2 * len(c.positions)))

    def bench_report(self, records, fmt: str = "json") -> str:
        """emit_report (src/bench.cpp:329-369) over BenchRecord dicts
        {task, n, depth, threads, seconds, [speedup], params}."""
        arr, keep = abi.pack_bench_records(records)
        n = ct.c_int64()
        f = 1 if fmt == "csv" else 0
        self.check(self._fn("bench_report")(arr, len(records), f, None, 0, ct.byref(n)))
        buf = ct.create_string_buffer(n.value + 1)
        self.check(self._fn("bench_report")(arr, len(records), f, buf, n.value + 1, ct.byref(n)))
        del keep
        return buf.value.decode()

    def channel_inverse(self, c):
        """-> (inverse or None when singular, condition) of the channel's
        superoperator, as gradient_mixed inverts it."""
        d = 1 << (2 * len(c.positions))
        out = np.zeros(d * d, dtype=np.complex128)
        cond, sing = ct.c_double(), ct.c_int32()
        p = pack_ops([c])
        self.check(self._fn("channel_inverse")(p.arr, out.ctypes.data_as(c128_p), ct.byref(cond), ct.byref(sing)))
        return (None if sing.value else out), cond.value
