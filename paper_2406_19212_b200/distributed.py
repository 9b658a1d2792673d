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
        self.swaps = 0              # exchange rounds
        self.swapped_bits = 0       # global<->local bit exchanges over all rounds
        self.bytes_exchanged = 0    # sent by this rank
        self.max_buffer_amps = 0    # largest single transfer buffer
        self.inflight_amps = 0      # most receive-buffer amplitudes in flight at once
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
    def _chunks(self, view, limit: int):
        """Index tuples that cut a (strided) view into pieces of at most
        `limit` elements: split the outermost dimension whose inner block
        fits, iterate over every index of the dimensions before it."""
        import itertools
        dims = list(view.shape)
        inner = 1
        d = len(dims)
        while d > 0 and inner * dims[d - 1] <= limit:
            inner *= dims[d - 1]
            d -= 1
        if d == 0:
            yield ()
            return
        step = max(1, limit // inner)
        for head in itertools.product(*[range(x) for x in dims[:d - 1]]):
            for a in range(0, dims[d - 1], step):
                yield head + (slice(a, min(dims[d - 1], a + step)),)

    def _swap_many(self, pairs) -> None:
        """Exchange k physical global bits with k local bits in one all-to-all
        round (pairs = [(global bit, local bit), ...], k <= g).

        Rank r with value a on the global bits G exchanges, for every b != a,
        its amplitudes whose local bits L equal b with the rank r' (G bits = b)
        amplitudes whose L bits equal a; those land in the slots with L bits
        = b. All 2^k - 1 partners are served by one grouped send/recv per
        chunk. Every transfer buffer is bounded: the receive buffers of one
        round in flight (two chunk generations x partners) hold at most
        `chunk_amps` amplitudes together, the send staging as much."""
        import torch
        pairs = sorted(pairs, key=lambda p: p[1])
        k = len(pairs)
        G = [gp - self.n_loc for gp, _ in pairs]
        L = [lp for _, lp in pairs]
        a = sum(((self.rank >> G[i]) & 1) << i for i in range(k))
        partners = []
        for b in range(1 << k):
            if b == a:
                continue
            r2 = self.rank
            for i in range(k):
                r2 = (r2 & ~(1 << G[i])) | (((b >> i) & 1) << G[i])
            partners.append((b, r2))
        per = max(1, self.chunk // (2 * len(partners)))  # two generations in flight
        # shard viewed with one dimension of size 2 per local bit in L
        # (ascending), rest dims in between: [hi, 2, mid_{k-1}, ..., 2, lo]
        shape = []
        prev = self.n_loc
        for l in reversed(L):
            shape += [1 << (prev - l - 1), 2]
            prev = l
        shape.append(1 << prev)

        def select(v, b):
            # index the "2" dims (positions 1, 3, ...) with b's bits (high L first)
            idx = []
            for j, l in enumerate(reversed(L)):
                bit = (b >> (k - 1 - j)) & 1
                idx += [slice(None), bit]
            return v[tuple(idx)]

        for shard in [self.local] + self.followers:
            v = shard.view(*shape)
            views = [(select(v, b), r2) for b, r2 in partners]
            slices = list(self._chunks(views[0][0], per))
            pending = []

            def finish(item):
                reqs, bufs = item
                for req in reqs:
                    req.wait()
                for (dst, sl), rbuf in bufs:
                    dst[sl] = torch.view_as_complex(rbuf).view(dst[sl].shape)

            for sl in slices:
                ops, bufs = [], []
                for dst, r2 in views:
                    sbuf = torch.view_as_real(dst[sl].contiguous()).reshape(-1)
                    rbuf = torch.empty_like(sbuf)
                    self.max_buffer_amps = max(self.max_buffer_amps, rbuf.numel() // 2)
                    if self.world > 1:
                        ops += [self.dist.P2POp(self.dist.isend, sbuf, r2),
                                self.dist.P2POp(self.dist.irecv, rbuf, r2)]
                    else:
                        rbuf.copy_(sbuf)
                    bufs.append(((dst, sl), rbuf.view(-1, 2)))
                    self.bytes_exchanged += sbuf.numel() * 8
                reqs = self.dist.batch_isend_irecv(ops) if ops else []
                pending.append((reqs, bufs))
                self.inflight_amps = max(self.inflight_amps,
                                         sum(rb.numel() // 2 for _, b in pending for _, rb in b))
                if len(pending) == 2:
                    finish(pending.pop(0))
            for item in pending:
                finish(item)
        # logical qubits on the exchanged physical bits trade places
        for gp, lp in pairs:
            x = self.log2phys.index(gp)
            y = self.log2phys.index(lp)
            self.log2phys[x], self.log2phys[y] = lp, gp
        self.swaps += 1
        self.swapped_bits += k

    def _swap(self, gpos: int, lpos: int) -> None:
        """Exchange physical global bit gpos (>= n_loc) with local bit lpos."""
        self._swap_many([(gpos, lpos)])

    def _bring_local(self, need_global, upcoming, avoid) -> None:
        """Swap the global physical bits `need_global` local in one round,
        together with every other global bit a mixing operation in
        `upcoming` (phys-bit sets, program order) needs, as long as free local
        bits remain. Local partners: bits not in `avoid` and unused by the
        upcoming operations, highest first (long contiguous runs)."""
        soon = set()
        for bits in upcoming:
            soon.update(bits)
        want = list(dict.fromkeys(need_global))
        for bits in upcoming:
            for b in bits:
                if b >= self.n_loc and b not in want:
                    want.append(b)
        free = [l for l in range(self.n_loc - 1, -1, -1) if l not in avoid and l not in soon]
        rest = [l for l in range(self.n_loc - 1, -1, -1) if l not in avoid and l in soon]
        pairs = []
        for gb in want:
            if free:
                pairs.append((gb, free.pop(0)))
            elif gb in need_global and rest:
                pairs.append((gb, rest.pop(0)))
        self._swap_many(pairs)

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
            need = [phys[b] for b in mix if phys[b] >= self.n_loc]
            if need:
                # one all-to-all round brings this gate's global mixing bits
                # local, plus those of the next gates while free local bits last
                self._flush(batch)
                upcoming = []
                for f in elems[idx + 1: idx + 1 + lookahead]:
                    fm = _mixing_bits(self._gate_matrix(f), len(f.positions))
                    upcoming.append([self.log2phys[f.positions[b] - 1] for b in fm])
                self._bring_local(need, upcoming, set(phys))
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
        need = [self.log2phys[q] for q in sorted(xy) if self.log2phys[q] >= self.n_loc]
        if need:
            cands = [b for b in range(self.n_loc - 1, -1, -1) if self.log2phys.index(b) not in xy]
            if len(cands) < len(need):
                raise UnsupportedError("expectation: too many X/Y qubits for the local shard")
            self._swap_many(list(zip(need, cands)))
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
                need = [phys[b] for b in sorted(mix) if phys[b] >= self.n_loc]
                if need:
                    self.engine.reverse_sweep(self, psi, steps, grads)
                    steps = []
                    upcoming = []
                    for f in reversed(elems[max(0, i - lookahead): i]):
                        fm = set(_mixing_bits(self.engine.gate_inverse(f), len(f.positions)))
                        for p_ in range(len(f.is_param)):
                            if f.is_param[p_]:
                                fm.update(_mixing_bits(self.engine.gate_derivative(f, p_), len(f.positions)))
                        upcoming.append([self.log2phys[f.positions[b] - 1] for b in sorted(fm)])
                    self._bring_local(need, upcoming, set(phys))
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
        import torch
        torch.cuda.current_stream().synchronize()  # swaps write the shard on torch's stream
        s = self._wrap(st)
        v = self.eng.norm(s) ** 2
        s.free()
        return v

    def local_expectation(self, st: ShardedState, op: PauliOperator) -> complex:
        import torch
        torch.cuda.current_stream().synchronize()
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
