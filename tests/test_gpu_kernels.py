"""GPU parity: gate/channel application through the C-ABI against the CPU
checker (the reference library compiled from /root/reference, oracle/_ref).

Cases restate the reference's kernel tests (tests/test_kernels.cpp:58-424).
Tolerances: amplitudes max-abs <= 1e-12 (BASELINE.json north_star); exact
permutations (X, CNOT, SWAP, Toffoli-free named swaps) bit-exact.
"""
import numpy as np
import pytest

from paper_2406_19212_b200 import circuits
from paper_2406_19212_b200.abi import (ChannelKind, Circuit, GateKind, IndexError_, TypeError_,
                                       ValidityError, make_gate, parametric_gate,
                                       standard_channel, standard_gate)

from helpers import (random_channel, random_density, random_gate, random_positions,
                     random_state, random_unitary)

pytestmark = pytest.mark.gpu
TOL = 1e-12


def both(dev, ref, amps, mixed=False):
    return dev.from_amplitudes(amps, mixed), ref.from_amplitudes(amps, mixed)


def test_textbook_actions(dev):
    # tests/test_kernels.cpp:58-75
    s = dev.pure_state(1)
    dev.apply_gate(s, standard_gate(GateKind.H, [1]))
    a = dev.download(s)
    assert np.allclose(a, [2 ** -0.5, 2 ** -0.5], atol=1e-15)
    t = dev.from_amplitudes(np.array([0, 1, 0, 0], dtype=complex))
    dev.apply_gate(t, standard_gate(GateKind.Cnot, [1, 2]))
    a = dev.download(t)
    assert a[3] == 1 and a[1] == 0
    u = dev.pure_state(2)
    with pytest.raises(IndexError_):
        dev.apply_gate(u, standard_gate(GateKind.X, [3]))
    with pytest.raises(ValidityError):
        dev.apply_gate(u, make_gate([1, 1], np.eye(4)))


@pytest.mark.parametrize("targets", [[1, 2], [2, 9], [9, 12], [12, 3], [14, 13], [1], [4], [5], [14]])
def test_dense_all_index_cases(dev, ref, targets):
    # tests/test_kernels.cpp:137-152 (BothLow / Mixed / BothHigh)
    rng = np.random.default_rng(42 + sum(targets))
    n = 14
    g = make_gate(targets, random_unitary(1 << len(targets), rng))
    amps = random_state(n, rng)
    d, r = both(dev, ref, amps)
    dev.apply_gate(d, g)
    ref.apply_gate(r, g)
    assert np.max(np.abs(dev.download(d) - ref.download(r))) <= TOL


def test_identity_gate_bit_exact(dev):
    rng = np.random.default_rng(4)
    amps = random_state(10, rng)
    s = dev.from_amplitudes(amps)
    dev.apply_gate(s, make_gate([3, 8], np.eye(4)))
    assert np.array_equal(dev.download(s), amps)


@pytest.mark.parametrize("kind", [GateKind.X, GateKind.Z, GateKind.S, GateKind.T, GateKind.Y,
                                  GateKind.H, GateKind.SqrtX, GateKind.SqrtY])
def test_named_1q(dev, ref, kind):
    rng = np.random.default_rng(8)
    n = 11
    for q in (1, 6, 11):
        amps = random_state(n, rng)
        d, r = both(dev, ref, amps)
        g = standard_gate(kind, [q])
        dev.apply_gate(d, g)
        ref.apply_gate(r, g)
        a, b = dev.download(d), ref.download(r)
        if kind == GateKind.X:
            assert np.array_equal(a, b)  # exact permutation
        assert np.max(np.abs(a - b)) <= TOL


@pytest.mark.parametrize("kind", [GateKind.CZ, GateKind.Cnot, GateKind.Swap, GateKind.ISwap])
def test_named_2q(dev, ref, kind):
    rng = np.random.default_rng(9)
    n = 11
    for pos in ([1, 2], [7, 3], [5, 11], [11, 1]):
        amps = random_state(n, rng)
        d, r = both(dev, ref, amps)
        g = standard_gate(kind, pos)
        dev.apply_gate(d, g)
        ref.apply_gate(r, g)
        a, b = dev.download(d), ref.download(r)
        if kind in (GateKind.Cnot, GateKind.Swap):
            assert np.array_equal(a, b)
        assert np.max(np.abs(a - b)) <= TOL


def test_three_qubit_dense_fallback(dev, ref):
    rng = np.random.default_rng(10)
    n = 11
    for g in (standard_gate(GateKind.Toffoli, [2, 9, 5]), standard_gate(GateKind.Fredkin, [10, 1, 6]),
              make_gate([3, 1, 7, 11], random_unitary(16, rng))):
        amps = random_state(n, rng)
        d, r = both(dev, ref, amps)
        dev.apply_gate(d, g)
        ref.apply_gate(r, g)
        assert np.max(np.abs(dev.download(d) - ref.download(r))) <= TOL


def test_random_gates_small_states(dev, ref):
    # tests/test_kernels.cpp:190-197, including states with < 8 bases
    rng = np.random.default_rng(21)
    for _ in range(60):
        n = int(rng.integers(2, 11))
        g = random_gate(n, rng)
        amps = random_state(n, rng)
        d, r = both(dev, ref, amps)
        dev.apply_gate(d, g)
        ref.apply_gate(r, g)
        assert np.max(np.abs(dev.download(d) - ref.download(r))) <= TOL


def test_norm_preserved_over_long_sequence(dev):
    # tests/test_kernels.cpp:199-207
    rng = np.random.default_rng(33)
    n = 8
    c = Circuit([random_gate(n, rng) for _ in range(1000)])
    s = dev.pure_state(n)
    dev.apply_circuit(c, s)
    assert abs(dev.norm(s) - 1.0) <= 1e-10


@pytest.mark.parametrize("fused", [True, False])
def test_circuit_matches_reference(dev, ref, fused):
    rng = np.random.default_rng(55)
    n = 13
    c = Circuit([random_gate(n, rng) for _ in range(200)])
    amps = random_state(n, rng)
    d, r = both(dev, ref, amps)
    dev.apply_circuit(c, d, fused=fused)
    ref.apply_circuit(c, r)
    assert np.max(np.abs(dev.download(d) - ref.download(r))) <= TOL


def test_apply_matrix_non_unitary(dev, ref):
    rng = np.random.default_rng(56)
    n = 9
    for m in (1, 2, 3, 4, 5):
        pos = random_positions(n, m, rng)
        mat = (rng.standard_normal((1 << m, 1 << m)) + 1j * rng.standard_normal((1 << m, 1 << m))) / 4
        amps = random_state(n, rng)
        d, r = both(dev, ref, amps)
        dev.apply_matrix(d, pos, mat)
        ref.apply_matrix(r, pos, mat)
        assert np.max(np.abs(dev.download(d) - ref.download(r))) <= TOL


# ---------------- density matrices ----------------
def test_mixed_gate_known_answers(dev):
    # tests/test_kernels.cpp:255-270
    dm = dev.mixed_state(1)
    dev.apply_gate(dm, standard_gate(GateKind.X, [1]))
    e = dev.download(dm)
    assert e[3] == 1 and e[0] == 0
    dh = dev.mixed_state(1)
    dev.apply_gate(dh, standard_gate(GateKind.H, [1]))
    assert np.allclose(dev.download(dh), 0.5, atol=1e-12)


def test_channel_known_answers(dev):
    # tests/test_kernels.cpp:290-309
    dm = dev.mixed_state(1)
    dev.apply_channel(dm, standard_channel(ChannelKind.Depolarizing, 1, 1.0))
    e = dev.download(dm)
    assert abs(e[0] - 0.5) < 1e-13 and abs(e[3] - 0.5) < 1e-13
    plus = dev.from_amplitudes(np.array([0.5, 0.5, 0.5, 0.5], dtype=complex), mixed=True)
    gamma = 0.4
    dev.apply_channel(plus, standard_channel(ChannelKind.PhaseDamping, 1, gamma))
    e = dev.download(plus)
    assert abs(e[2] - 0.5 * np.sqrt(1 - gamma)) < 1e-13 and abs(e[0] - 0.5) < 1e-13
    with pytest.raises(IndexError_):
        dev.apply_channel(dm, standard_channel(ChannelKind.PhaseDamping, 3, 0.1))
    with pytest.raises(TypeError_):
        dev.apply_channel(dev.pure_state(2), standard_channel(ChannelKind.PhaseDamping, 1, 0.1))


def test_interleaved_gates_and_channels(dev, ref):
    # tests/test_kernels.cpp:311-344
    rng = np.random.default_rng(90)
    n = 4
    for _ in range(6):
        elems = []
        for _ in range(12):
            if rng.integers(2) == 0:
                elems.append(random_gate(n, rng, max_targets=2))
            else:
                elems.append(random_channel(n, rng))
        elems.append(circuits.make_channel([1, 3], circuits.depolarizing2_kraus(0.3)))
        c = Circuit(elems)
        rho = random_density(n, rng)
        d, r = both(dev, ref, rho, mixed=True)
        dev.apply_circuit(c, d)
        ref.apply_circuit(c, r)
        assert np.max(np.abs(dev.download(d) - ref.download(r))) <= TOL
        assert abs(dev.trace(d) - 1) <= 1e-10


def test_trace_drift(dev):
    # tests/test_kernels.cpp:346-361
    rng = np.random.default_rng(13)
    n = 3
    elems = [standard_gate(GateKind.H, [1]), standard_gate(GateKind.Cnot, [1, 2])]
    elems += [random_channel(n, rng) for _ in range(100)]
    dm = dev.mixed_state(n)
    dev.apply_circuit(Circuit(elems), dm)
    assert abs(dev.trace(dm) - 1) <= 1e-10


# ---------------- bilinear form / reverse step ----------------
def test_bilinear_form(dev, ref):
    # tests/test_kernels.cpp:363-387
    rng = np.random.default_rng(101)
    n = 7
    for _ in range(10):
        m = int(rng.integers(1, 4))
        pos = random_positions(n, m, rng)
        local = (rng.uniform(-1, 1, (1 << m, 1 << m)) + 1j * rng.uniform(-1, 1, (1 << m, 1 << m)))
        bra, ket = random_state(n, rng), random_state(n, rng)
        db, dk = both(dev, ref, bra)[0], dev.from_amplitudes(ket)
        rb, rk = ref.from_amplitudes(bra), ref.from_amplitudes(ket)
        got = dev.bilinear_form(db, dk, pos, local)
        want = ref.bilinear_form(rb, rk, pos, local)
        assert abs(got - want) <= 1e-12


def test_reverse_step(dev, ref):
    # tests/test_kernels.cpp:389-424 (+ multi-parameter and 4-position cases)
    rng = np.random.default_rng(202)
    n = 8
    for rep in range(12):
        if rep % 3 == 0:
            g = parametric_gate(GateKind.Ry, random_positions(n, 1, rng), 3 * rng.random(), True)
        elif rep % 3 == 1:
            g = parametric_gate(GateKind.Fsim, random_positions(n, 2, rng),
                                list(rng.uniform(-2, 2, 5)), [True] * 5)
        else:
            g = parametric_gate(GateKind.CRx, random_positions(n, 2, rng), 1.3, True)
        inv = ref.gate_inverse(g)
        dmats = [ref.gate_derivative(g, p) for p in range(len(g.params))]
        a, b = random_state(n, rng), random_state(n, rng)
        dphi, dpsi = dev.from_amplitudes(a), dev.from_amplitudes(b)
        rphi, rpsi = ref.from_amplitudes(a), ref.from_amplitudes(b)
        got = dev.reverse_step(dphi, dpsi, g.positions, inv, dmats)
        want = ref.reverse_step(rphi, rpsi, g.positions, inv, dmats)
        assert np.max(np.abs(np.array(got) - np.array(want))) <= 1e-13
        assert np.max(np.abs(dev.download(dphi) - ref.download(rphi))) <= 1e-14
        assert np.max(np.abs(dev.download(dpsi) - ref.download(rpsi))) <= 1e-14
    # 4 pseudo positions (DM superop locals)
    pos = random_positions(10, 4, rng)
    inv = random_unitary(16, rng)
    dmats = [random_unitary(16, rng) for _ in range(3)]
    a, b = random_state(10, rng), random_state(10, rng)
    dphi, dpsi = dev.from_amplitudes(a), dev.from_amplitudes(b)
    rphi, rpsi = ref.from_amplitudes(a), ref.from_amplitudes(b)
    got = dev.reverse_step(dphi, dpsi, pos, inv, dmats)
    want = ref.reverse_step(rphi, rpsi, pos, inv, dmats)
    assert np.max(np.abs(np.array(got) - np.array(want))) <= 1e-12


@pytest.mark.parametrize("tile_bits,fuse", [("8", "2"), ("10", "0"), ("12", "2"), ("7", "1")])
def test_fused_planner_variants(dev, ref, monkeypatch, tile_bits, fuse):
    """Stage planning / block fusion under several tile sizes against the
    reference: random named, parametric and generic gates incl. controls on
    bits outside the tile."""
    monkeypatch.setenv("VQB_TILE_BITS", tile_bits)
    monkeypatch.setenv("VQB_TILE_BITS_REV", tile_bits)
    monkeypatch.setenv("VQB_FUSE_QUBITS", fuse)
    rng = np.random.default_rng(int(tile_bits) * 7 + int(fuse))
    n = 15
    c = Circuit([random_gate(n, rng) for _ in range(300)])
    amps = random_state(n, rng)
    d, r = both(dev, ref, amps)
    dev.apply_circuit(c, d)
    ref.apply_circuit(c, r)
    assert np.max(np.abs(dev.download(d) - ref.download(r))) <= TOL
    w = circuits.config2(n=12, p=2)
    loss, g = dev.gradient_pure(w.observable, w.circuit, dev.pure_state(12))
    rloss, rg = ref.gradient_pure(w.observable, w.circuit, ref.pure_state(12))
    assert abs(loss - rloss) <= 1e-10 * abs(rloss)
    assert np.max(np.abs(g - rg)) <= 1e-10 * np.max(np.abs(rg))
    w = circuits.config3(n=4, layers=1)
    loss, g = dev.gradient_mixed(w.observable, w.circuit, dev.mixed_state(4))
    rloss, rg = ref.gradient_mixed(w.observable, w.circuit, ref.mixed_state(4))
    assert abs(loss - rloss) <= 1e-10 * abs(rloss)
    assert np.max(np.abs(g - rg)) <= 1e-10 * np.max(np.abs(rg))


@pytest.mark.parametrize("mixed", [False, True])
def test_apply_circuit_copy_batch(dev, ref, mixed):
    """vqb_apply_circuit_copy_batch (pipelined apply_circuit_copy over host
    states, circuit.hpp:132-146): every output equals the reference's
    apply_circuit on that input; more jobs than device slots, so slots are
    reused."""
    rng = np.random.default_rng(17)
    if mixed:
        n = 6
        w = circuits.config3(n=n, layers=1)
        ins = [random_density(n, rng) for _ in range(5)]
    else:
        n = 14
        w = circuits.config1(rows=2, cols=7, cycles=4)
        ins = [random_state(n, rng) for _ in range(5)]
    outs = [np.empty_like(x) for x in ins]
    dev.apply_circuit_copy_batch(w.circuit, n, ins, outs, mixed=mixed)
    for x, y in zip(ins, outs):
        r = ref.from_amplitudes(x, mixed)
        ref.apply_circuit(w.circuit, r)
        assert np.max(np.abs(y - ref.download(r))) <= TOL
