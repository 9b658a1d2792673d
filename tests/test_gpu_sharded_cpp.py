"""GPU: the single-process multi-device sharded state (vqb_sharded_*,
csrc/sharded.cu) against the unsharded reference. This pool has one GPU per
box, so the P shards live on device 0 (devices = [0] * P): the exchange
kernels then read and write the peer shard through ordinary device pointers
— the same kernels and host logic as across NVLink peers, without the link.
Checks: whole state (canonical order, max-abs 1e-12) after random circuits
with mixing, controlled and diagonal gates on global qubits; expectation
values with X/Y factors on global qubits; norm; bit-exact permutations;
multi-bit all-to-all rounds."""
import numpy as np
import pytest

from paper_2406_19212_b200 import circuits
from paper_2406_19212_b200.abi import Circuit, GateKind, PauliTerm, parametric_gate, standard_gate

from helpers import random_gate, random_operator, random_state

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("P,n", [(2, 14), (4, 15), (8, 16)])
def test_sharded_random_circuit(dev, ref, P, n):
    rng = np.random.default_rng(100 + P)
    gates = [random_gate(n, rng) for _ in range(200)]
    top = n
    gates += [standard_gate(GateKind.H, [top]), standard_gate(GateKind.Cnot, [top, 1]),
              standard_gate(GateKind.Cnot, [2, top - 1]), parametric_gate(GateKind.Rz, [top], 0.7, True),
              parametric_gate(GateKind.Fsim, [top - 2, top], [0.3, 0.2, 0.1, 0.0, 0.4], [False] * 5),
              standard_gate(GateKind.CZ, [top, top - 1]), standard_gate(GateKind.Toffoli, [top, top - 1, 3])]
    c = Circuit(gates)
    psi = random_state(n, rng)
    sh = dev.sharded(n, [0] * P)
    sh.upload(psi)
    sh.apply_circuit(c)
    r = ref.from_amplitudes(psi)
    ref.apply_circuit(c, r)
    want = ref.download(r)
    assert np.max(np.abs(sh.download() - want)) <= 1e-12
    st = sh.stats()
    assert st["rounds"] > 0 and st["swapped_bits"] >= st["rounds"]
    assert abs(sh.norm() - 1) <= 1e-12
    op = random_operator(n, 10, rng)
    op.add_term(PauliTerm([(n, "x"), (n - 1, "y"), (1, "z")], 0.3))  # X/Y on global qubits
    log_before = sh.stats()["log2phys"]
    assert abs(sh.expectation(op) - ref.expectation(op, r)) <= 1e-12
    assert sh.stats()["log2phys"] == log_before  # partner shards read in place: no exchange
    assert np.max(np.abs(sh.download() - want)) <= 1e-12
    sh.free()


def test_sharded_rqc_multi_bit_rounds(dev, ref):
    """Config-1 family from |0...0>: the H-like layer on the top qubits brings
    all three global bits local in one round."""
    w = circuits.config1(rows=3, cols=5, cycles=10)
    sh = dev.sharded(15, [0] * 8)
    sh.apply_circuit(w.circuit)
    r = ref.pure_state(15)
    ref.apply_circuit(w.circuit, r)
    assert np.max(np.abs(sh.download() - ref.download(r))) <= 1e-12
    st = sh.stats()
    assert st["swapped_bits"] > st["rounds"]  # some rounds moved several bits
    sh.free()


def test_sharded_permutations_bit_exact(dev, ref):
    n = 14
    rng = np.random.default_rng(5)
    gates = []
    for _ in range(150):
        q = [int(x) + 1 for x in rng.choice(n, size=3, replace=False)]
        k = int(rng.integers(3))
        gates.append(standard_gate([GateKind.X, GateKind.Cnot, GateKind.Swap][k], q[:[1, 2, 2][k]]))
    psi = random_state(n, rng)
    sh = dev.sharded(n, [0] * 4)
    sh.upload(psi)
    sh.apply_circuit(Circuit(gates))
    r = ref.from_amplitudes(psi)
    ref.apply_circuit(Circuit(gates), r)
    assert np.array_equal(sh.download(), ref.download(r))
    sh.free()


def test_sharded_errors(dev):
    from paper_2406_19212_b200.abi import SizeError, TypeError_, UnsupportedError, standard_channel, ChannelKind
    with pytest.raises(UnsupportedError):
        dev.sharded(14, [0, 0, 0])  # not a power of two
    with pytest.raises(SizeError):
        dev.sharded(12, [0, 0])  # fewer than 12 local qubits
    sh = dev.sharded(13, [0, 0])
    with pytest.raises(TypeError_):
        sh.apply_circuit(Circuit([standard_channel(ChannelKind.Depolarizing, 1, 0.1)]))
    sh.free()


def test_sharded_dump_byte_identical(dev, ref, tmp_path):
    """vqb_sharded_save after swaps = the reference's save_state of the same
    state (io.hpp:56-82) byte for byte; loading it back restores the state."""
    w = circuits.config1(rows=3, cols=5, cycles=6)
    sh = dev.sharded(15, [0] * 4)
    sh.apply_circuit(w.circuit)
    assert sh.stats()["rounds"] > 0
    a = str(tmp_path / "sharded.vqcs")
    sh.save(a)
    assert sh.stats()["log2phys"] == list(range(15))  # canonical after the save
    r = ref.pure_state(15)
    ref.apply_circuit(w.circuit, r)
    b = str(tmp_path / "ref.vqcs")
    ref.save_state(r, b)
    da, db = open(a, "rb").read(), open(b, "rb").read()
    assert da[:13] == db[:13]  # header: magic, version, n, precision
    got = np.frombuffer(da[13:], dtype=np.complex128)
    assert np.max(np.abs(got - ref.download(r))) <= 1e-12
    # byte-identical to an unsharded dump of the same amplitudes
    s = dev.from_amplitudes(got)
    c = str(tmp_path / "plain.vqcs")
    dev.save_state(s, c)
    assert open(c, "rb").read() == da
    sh2 = dev.sharded(15, [0] * 4)
    assert sh2.load(a) == 2
    assert np.array_equal(sh2.download(), got)
    sh.free()
    sh2.free()


@pytest.mark.parametrize("P", [2, 4, 8])
def test_sharded_gradient_matches_reference(dev, ref, P):
    """gradient_pure on the sharded handle (QAOA: diagonal parametric steps
    on global qubits; hardware-efficient ansatz with a Heisenberg-like
    operator: X/Y factors and mixing parametric steps on global qubits)."""
    rng = np.random.default_rng(30 + P)
    n = 15
    cases = [circuits.config2(n=16, p=2), circuits.config0(n=n, layers=2)]
    for w in cases:
        op = w.observable if w is cases[0] else random_operator(w.num_qubits, 6, rng)
        sh = dev.sharded(w.num_qubits, [0] * P)
        loss, g = sh.gradient_pure(op, w.circuit)
        rl, rg = ref.gradient_pure(op, w.circuit, ref.pure_state(w.num_qubits))
        assert abs(loss - rl) <= 1e-10 * max(1.0, abs(rl))
        assert len(g) == len(rg)
        assert np.max(np.abs(g - rg)) <= 1e-10 * max(1.0, np.max(np.abs(rg)))
        back = sh.download()  # the reverse-swept Phi = s0 = |0...0>
        e0 = np.zeros_like(back)
        e0[0] = 1
        assert np.max(np.abs(back - e0)) <= 1e-10
        sh.free()
