"""Shared test fixtures: random states, unitaries, gates and operators in the
style of the reference's tests/oracles.hpp (:40-90, :236-282)."""
from __future__ import annotations

import math

import numpy as np

from paper_2406_19212_b200.abi import (ChannelKind, GateKind, PauliOperator, PauliTerm,
                                       make_channel, make_gate, parametric_gate, standard_channel,
                                       standard_gate)


def random_state(n: int, rng: np.random.Generator, mixed_pairs: int = 0) -> np.ndarray:
    """Unit-norm amplitudes with re/im ~ U[-1, 1) (oracles.hpp:45-62)."""
    v = (2 * rng.random(1 << n) - 1) + 1j * (2 * rng.random(1 << n) - 1)
    return (v / np.linalg.norm(v)).astype(np.complex128)


def random_density(n: int, rng: np.random.Generator, k: int = 2) -> np.ndarray:
    """Mixture of k random pure states, vec(rho) with entry (r, c) at r + c*2^n."""
    dim = 1 << n
    rho = np.zeros((dim, dim), dtype=np.complex128)
    for _ in range(k):
        psi = random_state(n, rng)
        rho += np.outer(psi, psi.conj()) / k
    return rho.flatten(order="F")


def random_unitary(d: int, rng: np.random.Generator) -> np.ndarray:
    z = (rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))) / math.sqrt(2)
    q, r = np.linalg.qr(z)
    return q * (np.diag(r) / np.abs(np.diag(r)))


def random_positions(n: int, m: int, rng: np.random.Generator) -> list:
    return [int(x) + 1 for x in rng.choice(n, size=m, replace=False)]


FIXED_1Q = [GateKind.X, GateKind.Y, GateKind.Z, GateKind.H, GateKind.S, GateKind.T,
            GateKind.SqrtX, GateKind.SqrtY]
FIXED_2Q = [GateKind.Swap, GateKind.ISwap, GateKind.CZ, GateKind.Cnot]
PARAM_1Q = [GateKind.Rx, GateKind.Ry, GateKind.Rz]
PARAM_2Q = [GateKind.CRx, GateKind.CRy, GateKind.CRz]


def random_gate(n: int, rng: np.random.Generator, max_targets: int = 3, active: bool = False):
    """Named fixed, parametric and Generic gates on random positions."""
    while True:
        choice = int(rng.integers(0, 7))
        if choice == 0:
            return standard_gate(FIXED_1Q[int(rng.integers(len(FIXED_1Q)))], random_positions(n, 1, rng))
        if choice == 1 and n >= 2 and max_targets >= 2:
            return standard_gate(FIXED_2Q[int(rng.integers(len(FIXED_2Q)))], random_positions(n, 2, rng))
        if choice == 2:
            return parametric_gate(PARAM_1Q[int(rng.integers(3))], random_positions(n, 1, rng),
                                   float(rng.uniform(-3, 3)), active)
        if choice == 3 and n >= 2 and max_targets >= 2:
            return parametric_gate(PARAM_2Q[int(rng.integers(3))], random_positions(n, 2, rng),
                                   float(rng.uniform(-3, 3)), active)
        if choice == 4 and n >= 2 and max_targets >= 2:
            return parametric_gate(GateKind.Fsim, random_positions(n, 2, rng),
                                   [float(x) for x in rng.uniform(-2, 2, 5)], [active] * 5)
        if choice == 5:
            m = int(rng.integers(1, min(max_targets, n) + 1))
            return make_gate(random_positions(n, m, rng), random_unitary(1 << m, rng))
        if choice == 6 and n >= 3 and max_targets >= 3:
            return standard_gate([GateKind.Toffoli, GateKind.Fredkin][int(rng.integers(2))],
                                 random_positions(n, 3, rng))


def random_channel(n: int, rng: np.random.Generator):
    kind = [ChannelKind.AmplitudeDamping, ChannelKind.PhaseDamping,
            ChannelKind.Depolarizing][int(rng.integers(3))]
    return standard_channel(kind, int(rng.integers(1, n + 1)), float(rng.uniform(0, 1)))


def random_operator(n: int, terms: int, rng: np.random.Generator, identity: bool = True):
    op = PauliOperator()
    if identity:
        op.add_term(PauliTerm([], complex(rng.uniform(-1, 1))))
    for _ in range(terms):
        k = int(rng.integers(1, min(n, 4) + 1))
        qs = random_positions(n, k, rng)
        op.add_term(PauliTerm([(q, "xyz"[int(rng.integers(3))]) for q in qs],
                              complex(rng.uniform(-1, 1), 0.0)))
    return op


def rel_err(a, b) -> float:
    a = np.asarray(a)
    b = np.asarray(b)
    den = max(float(np.max(np.abs(b))) if b.size else 0.0, 1e-300)
    return float(np.max(np.abs(a - b))) / den if b.size else 0.0


# ---------------------------------------------------------------- size-independent state checksums
# A state too large to compare whole (config 4: 2^33 amplitudes) is compared
# through a fixed sample of amplitudes and a few random projections
# P_j = sum_k w_j(k) a_k with weights hashed from the flat index k (SplitMix64
# finaliser, rng.hpp:31-36). A qubit relabelling, a transposed matrix or a
# misplaced superoperator changes every P_j by O(|a|·sqrt(2^n)) ~ O(1), while
# rounding moves them by ~1e-15 — so the projections pin the whole state.
NUM_PROJECTIONS = 4
_M64 = (1 << 64) - 1


def _mix64_np(k: np.ndarray) -> np.ndarray:
    z = k.astype(np.uint64) + np.uint64(0x9E3779B97F4A7C15)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def projection_weights(k0: int, count: int) -> np.ndarray:
    """[NUM_PROJECTIONS, count] float64 weights in [-0.5, 0.5) for indices
    k0 .. k0 + count - 1 (exactly representable: 16-bit fractions)."""
    with np.errstate(over="ignore"):
        z = _mix64_np(np.arange(k0, k0 + count, dtype=np.uint64))
    w = np.empty((NUM_PROJECTIONS, count), dtype=np.float64)
    for j in range(NUM_PROJECTIONS):
        w[j] = ((z >> np.uint64(16 * j)) & np.uint64(0xFFFF)).astype(np.float64) / 65536.0 - 0.5
    return w


def state_projections(eng, state, size: int, chunk: int = 1 << 24) -> np.ndarray:
    """Complex projections P_j of a state (any engine implementing
    state_download_range), streamed in chunks."""
    acc = np.zeros(NUM_PROJECTIONS, dtype=np.complex128)
    buf = np.empty(min(chunk, size), dtype=np.complex128)
    for k0 in range(0, size, chunk):
        c = min(chunk, size - k0)
        a = eng.download_range(state, k0, c, buf[:c])
        acc += projection_weights(k0, c) @ a
    return acc


def sample_indices(n_bits: int, count: int = 4096, seed: int = 12345) -> np.ndarray:
    """Sorted distinct flat indices: the first 64 plus `count` hashed ones."""
    with np.errstate(over="ignore"):
        z = _mix64_np(np.arange(count, dtype=np.uint64) + np.uint64(seed))
    idx = (z >> np.uint64(64 - n_bits)).astype(np.int64) if n_bits < 64 else z.astype(np.int64)
    return np.unique(np.concatenate([np.arange(min(64, 1 << n_bits)), idx]))


def sample_amplitudes(eng, state, idx: np.ndarray) -> np.ndarray:
    out = np.empty(len(idx), dtype=np.complex128)
    one = np.empty(1, dtype=np.complex128)
    # runs of consecutive indices in one call each
    i = 0
    while i < len(idx):
        j = i
        while j + 1 < len(idx) and idx[j + 1] == idx[j] + 1:
            j += 1
        out[i:j + 1] = eng.download_range(state, int(idx[i]), j - i + 1)
        i = j + 1
    del one
    return out


# Product-state projections: P_j = sum_k a_k prod_b f_b^(j)(bit b of k) with
# seeded unit-modulus factors f_b^(j)(0), f_b^(j)(1) -- the overlap of the
# state with a random (unnormalised) product state. Like the hashed
# projections they are O(1) for a random state and move by O(1) under a qubit
# relabelling, a transposed gate or a misplaced superoperator, but they
# contract bit by bit (no per-index hash), so a 2^33-amplitude state is
# checked in seconds on the device and in about a minute on the host.
def product_factors(n_bits: int) -> np.ndarray:
    """[n_bits, 2, NUM_PROJECTIONS] complex factors."""
    rng = np.random.default_rng(20240619)
    th = rng.uniform(0.0, 2.0 * np.pi, size=(n_bits, 2, NUM_PROJECTIONS))
    return np.exp(1j * th)


def _contract_chunk(a, F, lib):
    """sum over the chunk's bits (low bit first) -> [NUM_PROJECTIONS]."""
    cb = F.shape[0]
    t = a.reshape(-1, 2) @ F[0]                      # [2^(cb-1), J]
    for b in range(1, cb):
        t = lib.einsum("xij,ij->xj", t.reshape(-1, 2, NUM_PROJECTIONS), F[b])
    return t.reshape(NUM_PROJECTIONS)


def product_projections_host(eng, state, n_bits: int, chunk_bits: int = 24) -> np.ndarray:
    """P_j of a state of any engine implementing state_download_range."""
    F = product_factors(n_bits)
    cb = min(chunk_bits, n_bits)
    acc = np.zeros(NUM_PROJECTIONS, dtype=np.complex128)
    buf = np.empty(1 << cb, dtype=np.complex128)
    for c in range(1 << (n_bits - cb)):
        a = eng.download_range(state, c << cb, 1 << cb, buf)
        part = _contract_chunk(a, F[:cb], np)
        for b in range(cb, n_bits):
            part = part * F[b, (c >> (b - cb)) & 1]
        acc += part
    return acc


class _CudaArray:
    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": "<c16", "data": (ptr, False),
                                         "version": 3, "strides": None}


def device_view(eng, state):
    """Zero-copy complex128 torch view of a device state's amplitudes."""
    import ctypes as ct

    import torch
    p = ct.c_void_p()
    eng.check(eng._fn("state_device_ptr")(state.handle, ct.byref(p)))
    return torch.as_tensor(_CudaArray(p.value, state.size), device="cuda")


def product_projections_device(eng, state, n_bits: int, chunk_bits: int = 26) -> np.ndarray:
    """The same projections computed on the device (torch over the state's
    memory, chunk by chunk)."""
    import torch
    v = device_view(eng, state)
    torch.cuda.synchronize()
    F = torch.from_numpy(product_factors(n_bits)).to("cuda")
    cb = min(chunk_bits, n_bits)
    acc = torch.zeros(NUM_PROJECTIONS, dtype=torch.complex128, device="cuda")
    for c in range(1 << (n_bits - cb)):
        part = _contract_chunk(v[c << cb:(c + 1) << cb], F[:cb], torch)
        for b in range(cb, n_bits):
            part = part * F[b, (c >> (b - cb)) & 1]
        acc += part
    return acc.cpu().numpy()
