"""Seeded generators for the BASELINE.json configurations.

One generator per config builds the element list both sides consume (the
product through libvqcs_b200.so, the checker through oracle/), so parity runs
compare identical circuits. Randomness uses the reference's SplitMix64
(rng.hpp:38-64), `next_unit()` in (0, 1] (rng.hpp:51-54), Box-Muller
`next_normal_pair()` (rng.hpp:57-63) and `child_stream(seed, layer, qubit)`
(rng.hpp:68-71), restated here in exact 64-bit integer arithmetic.

Conventions BASELINE.json leaves open are pinned here once (SURVEY.md §8(d),
Appendix B) and recorded in DESIGN.md:
  * config 0/3 angles: one SplitMix64(seed) stream, theta = 2*pi*next_unit(),
    consumed in (layer, qubit, [Rz, Ry, Rz]) order;
  * config 1/4 couplers: A = horizontal (r,c)-(r,c+1) with c even, B = horizontal
    c odd, C = vertical (r,c)-(r+1,c) with r even, D = vertical r odd; cycle c
    uses pattern "ABCDCDAB"[c % 8]; qubit = 1 + r*cols + c;
  * config 1/4 one-qubit gate: child_stream(seed, cycle, qubit), first cycle
    uniform over {sqrtX, sqrtY, sqrtW}, later cycles uniform over the two gates
    that differ from the previous one; fSim angles from
    child_stream(seed, cycle, 1000 + coupler_index).next_normal_pair();
  * sqrtW = (1/sqrt2) [[e^{i pi/4}, -i], [1, e^{i pi/4}]] (Generic gate);
  * config 2: H on every qubit first; 3-regular graph by the stub-pairing model
    with rejection, driven by SplitMix64(seed); gamma_l, beta_l =
    pi * (1 - next_unit()) in [0, pi); ZZ phase as CNOT(i,j) Rz_j(2 gamma) CNOT(i,j);
    H_C = 1/2 sum_E (I - Z_i Z_j) as one identity term (|E|/2) + |E| ZZ terms;
  * config 3: 2q depolarizing Kraus K0 = sqrt(1 - 15p/16) I, K_ab = sqrt(p/16)
    sigma_a (x) sigma_b; amplitude damping after the CNOT block of each layer.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .abi import (ChannelKind, Circuit, GateKind, PauliOperator, PauliTerm, make_channel,
                  make_gate, parametric_gate, standard_channel, standard_gate, sum_z)

MASK64 = (1 << 64) - 1


def mix64(x: int) -> int:
    """rng.hpp:31-36."""
    x = (x + 0x9E3779B97F4A7C15) & MASK64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & MASK64
    return x ^ (x >> 31)


class SplitMix64:
    """rng.hpp:38-64."""

    def __init__(self, seed: int):
        self.state = seed & MASK64

    def next(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)

    def next_unit(self) -> float:
        """Uniform double in (0, 1]."""
        return float((self.next() >> 11) + 1) * (2.0 ** -53)

    def next_normal_pair(self):
        u1 = self.next_unit()
        u2 = self.next_unit()
        r = math.sqrt(-2.0 * math.log(u1))
        a = 2.0 * math.pi * u2
        return r * math.cos(a), r * math.sin(a)


def child_stream(seed: int, layer: int, qubit: int) -> SplitMix64:
    """rng.hpp:68-71."""
    return SplitMix64(mix64(mix64(mix64(seed) ^ layer) ^ ((qubit << 20 | qubit) & MASK64)))


SQRT_W = (1 / math.sqrt(2)) * np.array(
    [[np.exp(1j * math.pi / 4), -1j], [1.0, np.exp(1j * math.pi / 4)]], dtype=np.complex128)


def sqrt_w_gate(q: int):
    return make_gate([q], SQRT_W)


@dataclass
class Workload:
    name: str
    circuit: Circuit
    num_qubits: int
    mixed: bool = False
    observable: PauliOperator | None = None
    seed: int = 0
    extra: dict | None = None


# ---------------- config 0: hardware-efficient ansatz ----------------
def hea_circuit(n: int, layers: int, seed: int = 0) -> Circuit:
    rng = SplitMix64(seed)
    c = Circuit()
    for _ in range(layers):
        for q in range(1, n + 1):
            for kind in (GateKind.Rz, GateKind.Ry, GateKind.Rz):
                c.push_back(parametric_gate(kind, [q], 2.0 * math.pi * rng.next_unit(), True))
        for q in range(1, n):
            c.push_back(standard_gate(GateKind.Cnot, [q, q + 1]))
    return c


def config0(n: int = 20, layers: int = 10, seed: int = 0) -> Workload:
    return Workload("hea20_adjoint" if (n, layers) == (20, 10) else f"hea{n}x{layers}",
                    hea_circuit(n, layers, seed), n, False, sum_z(n), seed)


# ---------------- configs 1 and 4: random circuits on a grid ----------------
def grid_couplers(rows: int, cols: int):
    """-> dict letter -> list of (q1, q2) (1-based)."""
    q = lambda r, c: 1 + r * cols + c  # noqa: E731
    pats = {"A": [], "B": [], "C": [], "D": []}
    for r in range(rows):
        for c in range(cols - 1):
            pats["A" if c % 2 == 0 else "B"].append((q(r, c), q(r, c + 1)))
    for r in range(rows - 1):
        for c in range(cols):
            pats["C" if r % 2 == 0 else "D"].append((q(r, c), q(r + 1, c)))
    return pats


def rqc_circuit(rows: int, cols: int, cycles: int, seed: int = 0) -> Circuit:
    n = rows * cols
    pats = grid_couplers(rows, cols)
    order = "ABCDCDAB"
    coupler_index = {}
    for letter in "ABCD":
        for pair in pats[letter]:
            coupler_index[pair] = len(coupler_index)
    prev = [None] * (n + 1)
    c = Circuit()
    for cyc in range(cycles):
        for qb in range(1, n + 1):
            s = child_stream(seed, cyc, qb)
            u = s.next_unit()
            if prev[qb] is None:
                choice = min(int(u * 3.0), 2)
            else:
                others = [g for g in (0, 1, 2) if g != prev[qb]]
                choice = others[min(int(u * 2.0), 1)]
            prev[qb] = choice
            if choice == 0:
                c.push_back(standard_gate(GateKind.SqrtX, [qb]))
            elif choice == 1:
                c.push_back(standard_gate(GateKind.SqrtY, [qb]))
            else:
                c.push_back(sqrt_w_gate(qb))
        for pair in pats[order[cyc % 8]]:
            s = child_stream(seed, cyc, 1000 + coupler_index[pair])
            z1, z2 = s.next_normal_pair()
            theta = math.pi / 2 + 0.05 * z1
            phi = math.pi / 6 + 0.05 * z2
            c.push_back(parametric_gate(GateKind.Fsim, list(pair), [theta, phi, 0.0, 0.0, 0.0],
                                        [False] * 5))
    return c


def config1(rows: int = 4, cols: int = 7, cycles: int = 20, seed: int = 0) -> Workload:
    name = "rqc28_4x7_20cyc" if (rows, cols, cycles) == (4, 7, 20) else \
        f"rqc{rows * cols}_{rows}x{cols}_{cycles}cyc"
    return Workload(name, rqc_circuit(rows, cols, cycles, seed), rows * cols, seed=seed)


CONFIG4_GRIDS = {1: (3, 11), 2: (2, 17), 4: (5, 7), 8: (6, 6)}


def config4(num_gpus: int = 1, cycles: int = 14, seed: int = 0) -> Workload:
    rows, cols = CONFIG4_GRIDS[num_gpus]
    w = config1(rows, cols, cycles, seed)
    w.name = f"rqc{rows * cols}_{rows}x{cols}_{cycles}cyc_{num_gpus}gpu"
    return w


# ---------------- config 2: QAOA MaxCut ----------------
def random_regular_graph(n: int, degree: int, seed: int):
    rng = SplitMix64(seed)
    while True:
        stubs = [v for v in range(1, n + 1) for _ in range(degree)]
        for i in range(len(stubs) - 1, 0, -1):  # Fisher-Yates
            j = rng.next() % (i + 1)
            stubs[i], stubs[j] = stubs[j], stubs[i]
        edges = set()
        ok = True
        for k in range(0, len(stubs), 2):
            a, b = stubs[k], stubs[k + 1]
            if a == b or (min(a, b), max(a, b)) in edges:
                ok = False
                break
            edges.add((min(a, b), max(a, b)))
        if ok:
            return sorted(edges)


def qaoa_circuit(n: int, p: int, seed: int = 0):
    edges = random_regular_graph(n, 3, seed)
    rng = SplitMix64(seed ^ 0x5AA0)
    gammas = [math.pi * (1.0 - rng.next_unit()) for _ in range(p)]
    betas = [math.pi * (1.0 - rng.next_unit()) for _ in range(p)]
    c = Circuit()
    for q in range(1, n + 1):
        c.push_back(standard_gate(GateKind.H, [q]))
    for layer in range(p):
        for (i, j) in edges:
            c.push_back(standard_gate(GateKind.Cnot, [i, j]))
            c.push_back(parametric_gate(GateKind.Rz, [j], 2.0 * gammas[layer], True))
            c.push_back(standard_gate(GateKind.Cnot, [i, j]))
        for q in range(1, n + 1):
            c.push_back(parametric_gate(GateKind.Rx, [q], 2.0 * betas[layer], True))
    op = PauliOperator()
    op.add_term(PauliTerm([], 0.5 * len(edges)))
    for (i, j) in edges:
        op.add_term(PauliTerm([(i, "z"), (j, "z")], -0.5))
    return c, op, edges, gammas, betas


def qaoa_tied_gradients(per_gate: np.ndarray, n: int, num_edges: int, p: int) -> np.ndarray:
    """Chain rule for the tied QAOA parameters: d/dgamma_l = 2 sum_edges g(Rz),
    d/dbeta_l = 2 sum_qubits g(Rx). Returns [gamma_0..gamma_{p-1}, beta_0..]."""
    per = num_edges + n
    g = np.asarray(per_gate).reshape(p, per)
    return np.concatenate([2.0 * g[:, :num_edges].sum(axis=1), 2.0 * g[:, num_edges:].sum(axis=1)])


def config2(n: int = 30, p: int = 8, seed: int = 0) -> Workload:
    c, op, edges, gammas, betas = qaoa_circuit(n, p, seed)
    return Workload("qaoa30_p8" if (n, p) == (30, 8) else f"qaoa{n}_p{p}", c, n, False, op, seed,
                    {"edges": edges, "gammas": gammas, "betas": betas, "p": p})


# ---------------- config 3: noisy variational circuit on a density matrix ----------------
PAULI = {
    "i": np.eye(2, dtype=np.complex128),
    "x": np.array([[0, 1], [1, 0]], dtype=np.complex128),
    "y": np.array([[0, -1j], [1j, 0]], dtype=np.complex128),
    "z": np.array([[1, 0], [0, -1]], dtype=np.complex128),
}


def depolarizing2_kraus(p: float):
    ks = []
    for a in "ixyz":
        for b in "ixyz":
            # kron(high = second qubit, low = first qubit) in the local order
            op = np.kron(PAULI[b], PAULI[a])
            w = math.sqrt(1 - 15 * p / 16) if (a, b) == ("i", "i") else math.sqrt(p / 16)
            ks.append(w * op)
    return ks


def noisy_circuit(n: int, layers: int, p1: float = 1e-3, p2: float = 1e-2, gamma: float = 1e-3,
                  seed: int = 0) -> Circuit:
    rng = SplitMix64(seed)
    k2 = depolarizing2_kraus(p2)
    c = Circuit()
    for _ in range(layers):
        for q in range(1, n + 1):
            for kind in (GateKind.Rz, GateKind.Ry, GateKind.Rz):
                c.push_back(parametric_gate(kind, [q], 2.0 * math.pi * rng.next_unit(), True))
                c.push_back(standard_channel(ChannelKind.Depolarizing, q, p1))
        for q in range(1, n):
            c.push_back(standard_gate(GateKind.Cnot, [q, q + 1]))
            c.push_back(make_channel([q, q + 1], k2))
        for q in range(1, n + 1):
            c.push_back(standard_channel(ChannelKind.AmplitudeDamping, q, gamma))
    return c


def config3(n: int = 15, layers: int = 6, seed: int = 0) -> Workload:
    return Workload("noisy15_dm_6l" if (n, layers) == (15, 6) else f"noisy{n}_dm_{layers}l",
                    noisy_circuit(n, layers, seed=seed), n, True, sum_z(n), seed)


def touched_fraction(e) -> float:
    """Fraction of amplitudes a gate may change (SURVEY.md §8(d) touched-amplitude
    rule, mirroring the reference fast paths kernels.hpp:378-425)."""
    from .abi import GateOp
    if isinstance(e, GateOp):
        if e.kind in (GateKind.Cnot, GateKind.Swap, GateKind.Z, GateKind.S, GateKind.T):
            return 0.5
        if e.kind == GateKind.CZ:
            return 0.25
    return 1.0
