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
