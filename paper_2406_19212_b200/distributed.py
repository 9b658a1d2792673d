"""Sharded state vector over P = 2^g ranks (no reference
analogue — the reference is single-address-space, so its unsharded result is
the oracle).

Layout: physical bit positions 0..n_loc-1 are local (the rank's shard holds
2^n_loc amplitudes), positions n_loc..n-1 are global: rank r owns the
amplitudes whose global bits equal r. A logical->physical qubit map starts as
the identity and changes only through global<->local swaps.

Execution of a circuit (``ShardedState.apply_circuit``):
  * each gate is mapped to physical bits and analysed into mixing bits (the
    matrix couples them) and condition bits (block diagonal in them);
  * a mixing bit on a global position triggers a swap with a local position
    the gate does not use (pairwise exchange of half the shard with rank
    r XOR 2^j, in chunks, over torch.distributed: NCCL on GPUs, gloo in the CPU
    tests); the qubit map is updated, no data moves for the other ranks' bits;
  * condition bits on global positions are fixed to the rank's bit values on
    the host: the gate is replaced by its sub-matrix on the local positions
    (controls on global qubits and diagonal phases need no communication);
  * consecutive local gates are batched into one ``apply_circuit`` call of the
    local engine, i.e. one fused-executor run on the shard.

Reductions (norm, Z-string expectations): rank-local partials + one
all-reduce. ``gather`` returns the full state in the canonical (logical) order,
un-permuting the qubit map bit-exactly.

Adjoint gradients (``gradient_pure``, Algorithm 2 of autodiff.hpp:95-156):
the forward pass and the loss as above; the costate Psi = H|Phi> is built per
rank (Z factors on global qubits fold into a rank sign, X/Y factors are
swapped local first); Psi is a second shard that follows every swap of Phi (one
qubit map for both). The reverse loop walks the elements backwards; runs of
local steps (inverse and derivative matrices restricted on global condition
bits) go to the local engine as one batched reverse sweep (vqb_reverse_sweep,
the fused adjoint executor), a mixing bit on a global qubit swaps both shards
first. Each rank accumulates its partial gradient vector; one all-reduce sums
them at the end.

The local engine is any include/vqcs_b200.h implementation exposing
``wrap(tensor)``: the CUDA library on GPUs (``vqb_state_wrap`` over the shard's
device memory, no copy). Tests may pass a CPU engine.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable, List, Optional, Sequence

import numpy as np

from .abi import (ChannelOp, Circuit, GateKind, GateOp, PauliOperator, PauliTerm, UnsupportedError,
                  as_c128_array, make_gate)


def _mixing_bits(mat: np.ndarray, m: int) -> List[int]:
    """Local bit indices of an m-qubit column-major matrix that it mixes."""
    d = 1 << m
    M = mat.reshape(d, d, order="F")
    out = []
    for b in range(m):
        rows = np.arange(d)[:, None]
        cols = np.arange(d)[None, :]
        differ = ((rows ^ cols) >> b) & 1
        if np.any((differ == 1) & (M != 0)):
            out.append(b)
    return out


def _restrict(mat: np.ndarray, m: int, fixed: dict) -> np.ndarray:
    """Sub-matrix of an m-qubit matrix with local bits `fixed` (bit -> value)
    held constant (rows and columns); those bits must be non-mixing."""
    d = 1 << m
    M = mat.reshape(d, d, order="F")
    keep = [b for b in range(m) if b not in fixed]
    base = sum(v << b for b, v in fixed.items())
    idx = []
    for k in range(1 << len(keep)):
        i = base
        for q, b in enumerate(keep):
            if (k >> q) & 1:
                i |= 1 << b
        idx.append(i)
    idx = np.array(idx)
    return M[np.ix_(idx, idx)]


@dataclass
class LocalOp:
    positions: List[int]  # 1-based local physical positions
    matrix: np.ndarray    # column-major flattened


class ShardedState:
    """A pure n-qubit state sharded over the ranks of `group`."""

    def __init__(self, n: int, dist, engine, tensor, rank: int, world: int,
                 chunk_amps: int = 1 << 24):
        g = int(round(math.log2(world)))
        if 1 << g != world:
            raise UnsupportedError("world size must be a power of two")
        if n - g < 3:
            raise UnsupportedError("need at least 3 local qubits per rank")
        self.n, self.g, self.n_loc = n, g, n - g
        self.dist = dist
        self.engine = engine
        self.rank, self.world = rank, world
        self.local = tensor  # complex128 tensor of 2^n_loc amplitudes
        self.log2phys = list(range(n))  # logical qubit (0-based) -> physical bit
        self.chunk = chunk_amps
        self.followers: list = []  # extra shards (the adjoint costate) sharing the qubit map
        self.swaps = 0
        self.bytes_exchanged = 0
        self._gate_matrix = engine.gate_matrix

    # ---------------------------------------------------------------- init / io
    def set_zero(self) -> None:
        self.local.zero_()
        if self.rank == 0:
            self.local[0] = 1.0
        self.log2phys = list(range(self.n))

    def gather(self) -> Optional[np.ndarray]:
        """Full state in canonical order on rank 0 (None elsewhere)."""
        import torch
        # collectives move float64 views (gloo has no complex128)
        loc = torch.view_as_real(self.local.contiguous())
        parts = [torch.empty_like(loc) for _ in range(self.world)] if self.rank == 0 else None
        if self.world == 1:
            parts = [loc]
        else:
            self.dist.gather(loc, parts, dst=0)
        if self.rank != 0:
            return None
        phys = np.concatenate([torch.view_as_complex(p).cpu().numpy() for p in parts])  # physical order
        # amplitude with logical bits L sits at physical index P(L)
        idx = np.arange(1 << self.n, dtype=np.int64)
        pidx = np.zeros_like(idx)
        for q in range(self.n):
            pidx |= ((idx >> q) & 1) << self.log2phys[q]
        return phys[pidx]

    # ---------------------------------------------------------------- swaps
    def _swap(self, gpos: int, lpos: int) -> None:
        """Exchange physical global bit gpos (>= n_loc) with local bit lpos."""
        import torch
        j = gpos - self.n_loc
        partner = self.rank ^ (1 << j)
        mine = (self.rank >> j) & 1
        # local amplitudes with bit lpos == 1 - mine go to the partner, which
        # sends back its amplitudes with bit lpos == mine
        for shard in [self.local] + self.followers:
            v = shard.view(-1, 2, 1 << lpos)  # [hi, bit lpos, lo]
            send_half = v[:, 1 - mine, :]
            hi, lo = v.shape[0], v.shape[2]
            rows_per_chunk = max(1, self.chunk // lo)
            # two chunks in flight: chunk k+1's transfer overlaps chunk k's
            # copy into place (a chunk is overwritten only after its own send
            # completed; the send reads the shard directly when the half is
            # contiguous, lpos = top local bit)
            pending = []

            def finish(item):
                reqs, rbuf, a, b = item
                for req in reqs:
                    req.wait()
                send_half[a:b] = torch.view_as_complex(rbuf)

            for r0 in range(0, hi, rows_per_chunk):
                r1 = min(hi, r0 + rows_per_chunk)
                sbuf = torch.view_as_real(send_half[r0:r1].contiguous())
                rbuf = torch.empty_like(sbuf)
                reqs = []
                if self.world > 1:
                    ops = [self.dist.P2POp(self.dist.isend, sbuf, partner),
                           self.dist.P2POp(self.dist.irecv, rbuf, partner)]
                    reqs = self.dist.batch_isend_irecv(ops)
                pending.append((reqs, rbuf, r0, r1))
                self.bytes_exchanged += sbuf.numel() * 8
                if len(pending) == 2:
                    finish(pending.pop(0))
            for item in pending:
                finish(item)
        # logical qubits on the two physical bits trade places
        a = self.log2phys.index(gpos)
        b = self.log2phys.index(lpos)
        self.log2phys[a], self.log2phys[b] = lpos, gpos
        self.swaps += 1

    # ---------------------------------------------------------------- circuits
    def _flush(self, batch: List[LocalOp]) -> None:
        if not batch:
            return
        c = Circuit([make_gate([p for p in op.positions], op.matrix.reshape(-1)) for op in batch])
        self.engine.apply_local(self, c)
        batch.clear()

    def apply_circuit(self, circuit: Circuit, lookahead: int = 64) -> None:
        elems = list(circuit.elements)
        batch: List[LocalOp] = []
        for idx, e in enumerate(elems):
            if isinstance(e, ChannelOp):
                raise UnsupportedError("sharded states are pure; channels need a density matrix")
            mat = self._gate_matrix(e)
            m = len(e.positions)
            phys = [self.log2phys[p - 1] for p in e.positions]
            mix = _mixing_bits(mat, m)
            for b in mix:
                if phys[b] >= self.n_loc:
                    # bring it local: pick a local bit this gate does not use,
                    # preferring one not needed by the next gates
                    self._flush(batch)
                    soon = set()
                    for f in elems[idx + 1: idx + 1 + lookahead]:
                        soon.update(self.log2phys[p - 1] for p in f.positions)
                    cands = [l for l in range(self.n_loc - 1, -1, -1) if l not in phys]
                    pick = next((l for l in cands if l not in soon), cands[0])
                    self._swap(phys[b], pick)
                    phys = [self.log2phys[p - 1] for p in e.positions]
            fixed = {b: (self.rank >> (phys[b] - self.n_loc)) & 1
                     for b in range(m) if phys[b] >= self.n_loc}
            sub = _restrict(mat, m, fixed) if fixed else mat.reshape(1 << m, 1 << m, order="F")
            keep = [b for b in range(m) if b not in fixed]
            if not keep:  # fully global diagonal: a scalar phase on this rank
                ph = complex(sub[0, 0])
                if ph != 1:
                    batch.append(LocalOp([1], np.diag([ph, ph]).astype(np.complex128).reshape(-1, order="F")))
                continue
            if np.array_equal(sub, np.eye(sub.shape[0])):
                continue
            batch.append(LocalOp([phys[b] + 1 for b in keep],
                                 np.ascontiguousarray(sub.reshape(-1, order="F"))))
        self._flush(batch)

    # ---------------------------------------------------------------- reductions
    def _allreduce(self, x: complex) -> complex:
        if self.world == 1:
            return x
        import torch
        t = torch.tensor([x.real, x.imag], dtype=torch.float64, device=self.local.device)
        self.dist.all_reduce(t)
        return complex(float(t[0]), float(t[1]))

    def norm(self) -> float:
        local = float((self.local.abs() ** 2).sum()) if self.engine.host_reduce else \
            self.engine.local_norm_sq(self)
        return math.sqrt(self._allreduce(complex(local, 0)).real)

    def _local_operator(self, op: PauliOperator) -> PauliOperator:
        """This rank's share of a Pauli sum: X/Y factors made local (swaps),
        Z factors on global qubits folded into the rank's sign."""
        # every qubit carrying an X or Y factor in any term must be local; swap
        # global ones with local bits whose qubits carry no X/Y factor at all
        xy = {q - 1 for t in op.terms for q, l in t.factors if str(l).lower() in "xy"}
        for q in sorted(xy):
            if self.log2phys[q] >= self.n_loc:
                cands = [b for b in range(self.n_loc - 1, -1, -1)
                         if self.log2phys.index(b) not in xy]
                if not cands:
                    raise UnsupportedError("expectation: too many X/Y qubits for the local shard")
                self._swap(self.log2phys[q], cands[0])
        local_terms = []
        for t in op.terms:
            sign = 1
            factors = []
            for q, l in t.factors:
                p = self.log2phys[q - 1]
                if p >= self.n_loc:
                    if (self.rank >> (p - self.n_loc)) & 1:
                        sign = -sign
                else:
                    factors.append((p + 1, l))
            local_terms.append(PauliTerm(factors, sign * complex(t.coeff)))
        return PauliOperator(local_terms)

    def expectation(self, op: PauliOperator) -> complex:
        """Sum of Z-strings (any qubits, global ones fold into a sign) and, for
        X/Y factors, local qubits only (global X/Y factors are swapped local
        first)."""
        part = self.engine.local_expectation(self, self._local_operator(op))
        return self._allreduce(part)

    # ---------------------------------------------------------------- adjoint
    def _local_step(self, inv: np.ndarray, dmats: list, positions: list):
        """Restrict a reverse step to this rank: -> (local positions, inv,
        dmats) or None when it is the identity with no parameters."""
        m = len(positions)
        phys = [self.log2phys[p - 1] for p in positions]
        fixed = {b: (self.rank >> (phys[b] - self.n_loc)) & 1
                 for b in range(m) if phys[b] >= self.n_loc}

        def sub(mat):
            if fixed:
                return _restrict(mat, m, fixed)
            return np.asarray(mat).reshape(1 << m, 1 << m, order="F")

        keep = [b for b in range(m) if b not in fixed]
        inv_r = sub(inv)
        d_r = [sub(d) for d in dmats]
        if not keep:  # fully global diagonal: scalars on this rank (as a 1-bit op)
            eye = np.eye(2, dtype=np.complex128)
            return ([1], (inv_r[0, 0] * eye).reshape(-1, order="F"),
                    [(d[0, 0] * eye).reshape(-1, order="F") for d in d_r])
        if not d_r and np.array_equal(inv_r, np.eye(inv_r.shape[0])):
            return None
        return ([phys[b] + 1 for b in keep], np.ascontiguousarray(inv_r.reshape(-1, order="F")),
                [np.ascontiguousarray(d.reshape(-1, order="F")) for d in d_r])

    def gradient_pure(self, op: PauliOperator, circuit: Circuit, lookahead: int = 64):
        """gradient_pure (autodiff.hpp:95-156) on the shard: the state held
        now is s0; on return it holds the reverse-swept Phi (= s0 up to
        rounding). -> (loss, grads) on every rank."""
        import torch
        elems = list(circuit.elements)
        if any(isinstance(e, ChannelOp) for e in elems):
            raise UnsupportedError("gradient_pure: noisy circuits need gradient_mixed")
        base, total = [], 0
        for e in elems:  # parameter order: traversal, then in-gate (circuit.hpp:149-159)
            base.append(total)
            total += e.num_active_params()
        self.apply_circuit(circuit, lookahead)
        loss = self.expectation(op).real
        psi = torch.empty_like(self.local)
        self.engine.local_apply_operator(self, self._local_operator(op), psi)
        self.followers = [psi]
        grads = np.zeros(max(total, 1), dtype=np.float64)
        steps: list = []
        try:
            for i in range(len(elems) - 1, -1, -1):
                e = elems[i]
                inv = self.engine.gate_inverse(e)
                dmats = [self.engine.gate_derivative(e, p)
                         for p in range(len(e.is_param)) if e.is_param[p]]
                m = len(e.positions)
                mix = set(_mixing_bits(inv, m))
                for d in dmats:
                    mix.update(_mixing_bits(d, m))
                phys = [self.log2phys[p - 1] for p in e.positions]
                for b in sorted(mix):
                    if phys[b] >= self.n_loc:
                        self.engine.reverse_sweep(self, psi, steps, grads)
                        steps = []
                        soon = set()
                        for f in elems[max(0, i - lookahead): i]:
                            soon.update(self.log2phys[p - 1] for p in f.positions)
                        cands = [l for l in range(self.n_loc - 1, -1, -1) if l not in phys]
                        pick = next((l for l in cands if l not in soon), cands[0])
                        self._swap(phys[b], pick)
                        phys = [self.log2phys[p - 1] for p in e.positions]
                st = self._local_step(inv, dmats, list(e.positions))
                if st is not None:
                    steps.append((st[0], st[1], st[2], base[i]))
            self.engine.reverse_sweep(self, psi, steps, grads)
        finally:
            self.followers = []
        if self.world > 1:
            t = torch.from_numpy(grads).to(self.local.device)
            self.dist.all_reduce(t)
            grads = t.cpu().numpy()
        return loss, grads[:total]


class DeviceEngine:
    """Local engine on a GPU: the CUDA library over the shard's device memory."""

    host_reduce = False

    def __init__(self, eng):
        self.eng = eng
        self.gate_matrix = lambda g: eng.gate_matrix(g)

    def _wrap(self, st: ShardedState):
        import ctypes as ct
        from .engine import State
        h = ct.c_void_p()
        self.eng.check(self.eng._fn("state_wrap")(ct.c_void_p(st.local.data_ptr()), st.n_loc, 0,
                                                  ct.c_uint64(st.rank << st.n_loc), st.g,
                                                  ct.byref(h)))
        return State(self.eng, h, st.n_loc, False)

    def apply_local(self, st: ShardedState, c: Circuit) -> None:
        import torch
        torch.cuda.current_stream().synchronize()
        s = self._wrap(st)
        self.eng.apply_circuit(c, s)
        s.free()

    def local_norm_sq(self, st: ShardedState) -> float:
        s = self._wrap(st)
        v = self.eng.norm(s) ** 2
        s.free()
        return v

    def local_expectation(self, st: ShardedState, op: PauliOperator) -> complex:
        s = self._wrap(st)
        v = self.eng.expectation(op, s)
        s.free()
        return v

    def gate_inverse(self, g):
        return self.eng.gate_inverse(g)

    def gate_derivative(self, g, p):
        return self.eng.gate_derivative(g, p)

    def local_apply_operator(self, st: ShardedState, op: PauliOperator, out) -> None:
        """out <- op |shard> (apply_operator observables.hpp:216-237) on device."""
        import torch
        torch.cuda.current_stream().synchronize()
        src = self._wrap(st)
        dst = self._wrap_tensor(st, out)
        self.eng.check(self.eng._fn("apply_operator")(src.handle, dst.handle, *op.pack()[:2]))
        src.free()
        dst.free()

    def _wrap_tensor(self, st: ShardedState, tensor):
        import ctypes as ct
        from .engine import State
        h = ct.c_void_p()
        self.eng.check(self.eng._fn("state_wrap")(ct.c_void_p(tensor.data_ptr()), st.n_loc, 0,
                                                  ct.c_uint64(st.rank << st.n_loc), st.g,
                                                  ct.byref(h)))
        return State(self.eng, h, st.n_loc, False)

    def reverse_sweep(self, st: ShardedState, psi, steps, grads) -> None:
        if not steps:
            return
        import torch
        torch.cuda.current_stream().synchronize()
        a = self._wrap(st)
        b = self._wrap_tensor(st, psi)
        self.eng.reverse_sweep(a, b, steps, 2.0, grads)  # grads = 2 Re(acc) (autodiff.hpp:147-149)
        a.free()
        b.free()
