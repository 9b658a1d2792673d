"""GPU parity: observables, losses and adjoint gradients through the C-ABI
against the CPU checker (tests/test_observables.cpp, tests/test_autodiff.cpp).

Tolerance for expectations and gradients: ||d||_inf / ||ref||_inf <= 1e-10
(BASELINE.json north_star; SURVEY.md §7 — exactly-zero gradients come out near
1e-17 in the reference, so the check is normwise, not per element).
"""
import math

import numpy as np
import pytest

from paper_2406_19212_b200 import circuits
from paper_2406_19212_b200.abi import (ChannelKind, Circuit, GateKind, IndexError_,
                                       NonInvertibleChannelError, PauliOperator, PauliTerm,
                                       TypeError_, heisenberg_1d, parametric_gate,
                                       standard_channel, standard_gate, sum_z)

from helpers import random_density, random_gate, random_operator, random_state, rel_err

pytestmark = pytest.mark.gpu
RTOL = 1e-10


def z_on(q):
    return PauliOperator([PauliTerm([(q, "z")], 1.0)])


def test_expectation_known_answers(dev):
    # tests/test_observables.cpp:89-109
    assert dev.expectation(z_on(1), dev.pure_state(1)).real == pytest.approx(1.0)
    assert dev.expectation(heisenberg_1d(3), dev.pure_state(3)).real == pytest.approx(5.0)
    plus = dev.from_amplitudes(np.array([2 ** -0.5, 2 ** -0.5], dtype=complex))
    x1 = PauliOperator([PauliTerm([(1, "x")], 1.0)])
    assert dev.expectation(x1, plus).real == pytest.approx(1.0)
    with pytest.raises(IndexError_):
        dev.expectation(z_on(5), dev.pure_state(1))


def test_expectation_random(dev, ref):
    rng = np.random.default_rng(12)
    for n in (4, 9, 14):
        amps = random_state(n, rng)
        op = random_operator(n, 12, rng)
        got = dev.expectation(op, dev.from_amplitudes(amps))
        want = ref.expectation(op, ref.from_amplitudes(amps))
        assert abs(got - want) <= 1e-12


def test_expectation_mixed(dev, ref):
    # tests/test_observables.cpp:111-149
    mm = dev.from_amplitudes(np.array([0.5, 0, 0, 0.5], dtype=complex), mixed=True)
    assert abs(dev.expectation(z_on(1), mm)) < 1e-14
    one = dev.from_amplitudes(np.array([0, 0, 0, 1], dtype=complex), mixed=True)
    assert dev.expectation(z_on(1), one).real == pytest.approx(-1.0)
    rng = np.random.default_rng(9)
    for _ in range(5):
        n = 4
        rho = random_density(n, rng)
        op = random_operator(n, 6, rng)
        got = dev.expectation(op, dev.from_amplitudes(rho, mixed=True))
        want = ref.expectation(op, ref.from_amplitudes(rho, mixed=True))
        assert abs(got - want) <= 1e-12


def test_apply_operator(dev, ref):
    # tests/test_observables.cpp:151-179
    rng = np.random.default_rng(12)
    for _ in range(5):
        n = 6
        amps = random_state(n, rng)
        op = random_operator(n, 6, rng)
        got = dev.download(dev.apply_operator(op, dev.from_amplitudes(amps)))
        want = ref.download(ref.apply_operator(op, ref.from_amplitudes(amps)))
        assert np.max(np.abs(got - want)) <= 1e-12
        assert abs(np.vdot(amps, got) - dev.expectation(op, dev.from_amplitudes(amps))) <= 1e-10


@pytest.mark.parametrize("n", [8, 14, 18])
def test_apply_operator_z_diagonal(dev, ref, n):
    """The Z-diagonal fast path of apply_operator (one Z-string group with real
    coefficients: QAOA cost Hamiltonians, sums of Z): identity term, strings
    on low, middle (bits 5-7) and high qubits, against the reference."""
    rng = np.random.default_rng(n)
    amps = random_state(n, rng)
    terms = [PauliTerm([], 0.5)]
    for _ in range(30):
        k = int(rng.integers(1, 4))
        qs = sorted(set(int(q) + 1 for q in rng.choice(n, size=k, replace=False)))
        terms.append(PauliTerm([(q, "z") for q in qs], float(rng.standard_normal())))
    ops = [PauliOperator(terms), circuits.config2(n=n, p=1).observable, sum_z(n)]
    for op in ops:
        got = dev.download(dev.apply_operator(op, dev.from_amplitudes(amps)))
        want = ref.download(ref.apply_operator(op, ref.from_amplitudes(amps)))
        assert np.max(np.abs(got - want)) <= 1e-12


@pytest.mark.parametrize("theta", [0.0, 0.3, math.pi / 2, 1.9])
def test_rotated_qubit_gradient(dev, theta):
    # tests/test_autodiff.cpp:49-85
    c = Circuit([parametric_gate(GateKind.Rx, [1], theta, True)])
    loss, g = dev.gradient_pure(z_on(1), c, dev.pure_state(1))
    assert loss == pytest.approx(math.cos(theta), abs=1e-12)
    assert g[0] == pytest.approx(-math.sin(theta), abs=1e-10)


def test_no_active_params_and_channel_rejection(dev):
    fixed = Circuit([parametric_gate(GateKind.Rx, [1], 0.8, False), standard_gate(GateKind.H, [1])])
    loss, g = dev.gradient_pure(z_on(1), fixed, dev.pure_state(1))
    assert len(g) == 0
    noisy = Circuit([standard_channel(ChannelKind.Depolarizing, 1, 0.1)])
    with pytest.raises(TypeError_):
        dev.loss_pure(z_on(1), noisy, dev.pure_state(1))


@pytest.mark.parametrize("n,layers", [(6, 4), (12, 3), (20, 10)])
def test_config0_gradient(dev, ref, n, layers):
    w = circuits.config0(n=n, layers=layers)
    loss, g, res = dev.gradient_pure(w.observable, w.circuit, dev.pure_state(n), with_residual=True)
    rloss, rg = ref.gradient_pure(w.observable, w.circuit, ref.pure_state(n))
    assert abs(loss - rloss) <= RTOL * max(abs(rloss), 1e-300)
    assert rel_err(g, rg) <= RTOL
    assert res <= 1e-8
    if (n, layers) == (20, 10):  # golden values from the reference (tests/golden/config0_*.json)
        assert abs(loss - 0.19589280189123967) <= 1e-12


def test_multi_param_gates(dev, ref):
    # tests/test_autodiff.cpp:102-120
    c = Circuit([standard_gate(GateKind.H, [1]),
                 parametric_gate(GateKind.Fsim, [1, 2], [0.4, -0.3, 0.2, 0.7, -0.5], [True] * 5),
                 parametric_gate(GateKind.CRy, [2, 3], 0.9, True)])
    op = heisenberg_1d(3)
    loss, g = dev.gradient_pure(op, c, dev.pure_state(3))
    rloss, rg = ref.gradient_pure(op, c, ref.pure_state(3))
    assert len(g) == 6
    assert abs(loss - rloss) <= 1e-12
    assert rel_err(g, rg) <= RTOL


@pytest.mark.parametrize("n", [10, 15])
def test_random_circuit_gradient(dev, ref, n):
    rng = np.random.default_rng(77 + n)
    c = Circuit([random_gate(n, rng, active=True) for _ in range(120)])
    op = random_operator(n, 8, rng)
    amps = random_state(n, rng)
    loss, g = dev.gradient_pure(op, c, dev.from_amplitudes(amps))
    rloss, rg = ref.gradient_pure(op, c, ref.from_amplitudes(amps))
    assert abs(loss - rloss) <= RTOL * max(abs(rloss), 1e-12)
    assert rel_err(g, rg) <= RTOL


def test_qaoa_small_gradient(dev, ref):
    w = circuits.config2(n=10, p=3)
    loss, g = dev.gradient_pure(w.observable, w.circuit, dev.pure_state(10))
    rloss, rg = ref.gradient_pure(w.observable, w.circuit, ref.pure_state(10))
    assert abs(loss - rloss) <= RTOL * abs(rloss)
    assert rel_err(g, rg) <= RTOL
    tied = circuits.qaoa_tied_gradients(g, 10, len(w.extra["edges"]), 3)
    rtied = circuits.qaoa_tied_gradients(rg, 10, len(w.extra["edges"]), 3)
    assert rel_err(tied, rtied) <= RTOL


# ---------------- noisy ----------------
def test_noisy_known_answers(dev):
    # tests/test_autodiff.cpp:147-183
    p = 0.3
    for theta in (0.2, math.pi / 2, 2.4):
        c = Circuit([parametric_gate(GateKind.Rx, [1], theta, True),
                     standard_channel(ChannelKind.Depolarizing, 1, p)])
        loss, g = dev.gradient_mixed(z_on(1), c, dev.mixed_state(1))
        assert loss == pytest.approx((1 - p) * math.cos(theta), abs=1e-10)
        assert g[0] == pytest.approx(-(1 - p) * math.sin(theta), abs=1e-9)
        assert dev.loss_mixed(z_on(1), c, dev.mixed_state(1)) == pytest.approx(
            (1 - p) * math.cos(theta), abs=1e-10)


@pytest.mark.parametrize("n,layers", [(3, 2), (5, 2), (7, 1)])
def test_config3_gradient(dev, ref, n, layers):
    w = circuits.config3(n=n, layers=layers)
    loss, g = dev.gradient_mixed(w.observable, w.circuit, dev.mixed_state(n))
    rloss, rg = ref.gradient_mixed(w.observable, w.circuit, ref.mixed_state(n))
    assert abs(loss - rloss) <= RTOL * abs(rloss)
    assert rel_err(g, rg) <= RTOL


def test_pure_equals_mixed(dev):
    # tests/test_autodiff.cpp:200-210
    w = circuits.config0(n=4, layers=3)
    lp, gp = dev.gradient_pure(w.observable, w.circuit, dev.pure_state(4))
    lm, gm = dev.gradient_mixed(w.observable, w.circuit, dev.mixed_state(4))
    assert abs(lp - lm) <= 1e-8 and np.max(np.abs(gp - gm)) <= 1e-8


def test_non_invertible_channel(dev):
    # tests/test_autodiff.cpp:212-223
    c = Circuit([parametric_gate(GateKind.Rx, [1], 0.4, True),
                 standard_channel(ChannelKind.AmplitudeDamping, 1, 1.0)])
    with pytest.raises(NonInvertibleChannelError, match="AmplitudeDamping"):
        dev.gradient_mixed(z_on(1), c, dev.mixed_state(1))
    assert dev.loss_mixed(z_on(1), c, dev.mixed_state(1)) == pytest.approx(1.0)


def test_config0_full_gradient_and_rqc_roundtrip(dev):
    """Size-independent properties at full size: unitarity of the config-1
    circuit at 28 qubits (norm), and forward+inverse returns to |0>."""
    w = circuits.config1()
    s = dev.pure_state(28)
    dev.apply_circuit(w.circuit, s)
    assert abs(dev.norm(s) - 1.0) <= 1e-10


@pytest.mark.parametrize("executor", ["reg", "smem"])
def test_executors_agree_on_adjoint(dev, ref, monkeypatch, executor):
    """Both fused executors (register-resident and shared-memory) on the
    three gradient workloads at sizes where the register executor applies."""
    monkeypatch.setenv("VQB_EXECUTOR", executor)
    w = circuits.config2(n=14, p=2)
    loss, g = dev.gradient_pure(w.observable, w.circuit, dev.pure_state(14))
    rloss, rg = ref.gradient_pure(w.observable, w.circuit, ref.pure_state(14))
    assert abs(loss - rloss) <= RTOL * abs(rloss) and rel_err(g, rg) <= RTOL
    w = circuits.config3(n=7, layers=2)
    loss, g = dev.gradient_mixed(w.observable, w.circuit, dev.mixed_state(7))
    rloss, rg = ref.gradient_mixed(w.observable, w.circuit, ref.mixed_state(7))
    assert abs(loss - rloss) <= RTOL * abs(rloss) and rel_err(g, rg) <= RTOL
    w = circuits.config1(rows=3, cols=5, cycles=12)
    s = dev.pure_state(15)
    dev.apply_circuit(w.circuit, s)
    r = ref.pure_state(15)
    ref.apply_circuit(w.circuit, r)
    assert np.max(np.abs(dev.download(s) - ref.download(r))) <= 1e-12


@pytest.mark.parametrize("mode", ["block", "persistent"])
def test_specialised_kernels_match_reference(dev, ref, monkeypatch, mode):
    """Run-time specialised stage kernels (VQB_JIT=1, jit_rt.cuh) against the
    reference on forward programs with dense blocks, controls on tile and
    global bits, diagonal phases and per-register conditions."""
    from helpers import random_gate
    monkeypatch.setenv("VQB_JIT", "1")
    monkeypatch.setenv("VQB_JIT_MODE", mode)
    rng = np.random.default_rng(17)
    cases = [circuits.config1(rows=3, cols=5, cycles=12).circuit,
             circuits.config2(n=14, p=2).circuit,
             circuits.config0(n=15, layers=3).circuit,
             Circuit([random_gate(16, rng) for _ in range(300)])]
    for c in cases:
        n = max(q for e in c.elements for q in e.positions)
        n = max(n, 13)
        s = dev.pure_state(n)
        dev.apply_circuit(c, s)
        r = ref.pure_state(n)
        ref.apply_circuit(c, r)
        assert np.max(np.abs(dev.download(s) - ref.download(r))) <= 1e-12
    # a circuit's second call reuses the compiled kernels (new angles, same shape)
    w1, w2 = circuits.config2(n=14, p=2, seed=1), circuits.config2(n=14, p=2, seed=2)
    for w in (w1, w2):
        s = dev.pure_state(14)
        dev.apply_circuit(w.circuit, s)
        r = ref.pure_state(14)
        ref.apply_circuit(w.circuit, r)
        assert np.max(np.abs(dev.download(s) - ref.download(r))) <= 1e-12


@pytest.mark.parametrize("regs", ["8", "16"])
def test_specialised_adjoint_matches_reference(dev, ref, monkeypatch, regs):
    """Specialised adjoint kernels (VQB_JIT=1) for both register geometries:
    QAOA (folded diagonal parametric steps with register conditions), the
    hardware-efficient ansatz (1-qubit parametric steps + CNOT) and a noisy
    circuit (its 16x16 channel superoperators run in the specialised kernels
    too; only wide *parametric* steps would stay on the interpreter)."""
    monkeypatch.setenv("VQB_JIT", "1")
    monkeypatch.setenv("VQB_REV_REGS", regs)
    for w in (circuits.config2(n=14, p=2), circuits.config0(n=14, layers=3)):
        loss, g = dev.gradient_pure(w.observable, w.circuit, dev.pure_state(14))
        rloss, rg = ref.gradient_pure(w.observable, w.circuit, ref.pure_state(14))
        assert abs(loss - rloss) <= RTOL * abs(rloss) and rel_err(g, rg) <= RTOL
    w = circuits.config3(n=7, layers=2)
    loss, g = dev.gradient_mixed(w.observable, w.circuit, dev.mixed_state(7))
    rloss, rg = ref.gradient_mixed(w.observable, w.circuit, ref.mixed_state(7))
    assert abs(loss - rloss) <= RTOL * abs(rloss) and rel_err(g, rg) <= RTOL


@pytest.mark.parametrize("variant", [{}, {"VQB_JIT_DIAGRUN": "0"}, {"VQB_JIT_ACC": "1000"},
                                     {"VQB_JIT_LAZY": "0"}, {"VQB_PARALLEL_ADJOINT": "0"},
                                     {"VQB_JIT_GDIFF": "0"}, {"VQB_JIT_FACTOR": "1"},
                                     {"VQB_JIT_FACTOR": "1", "VQB_JIT_GDIFF": "0"},
                                     {"VQB_JIT_REDLANES": "1"}, {"VQB_JIT_REDLANES": "8"},
                                     {"VQB_JIT_DIRECT": "0"}, {"VQB_JIT_DOTPLAN": "0"},
                                     {"VQB_JIT_REDBATCH": "1"}, {"VQB_JIT_REDBATCH": "2"},
                                     {"VQB_MIXED_SPLIT": "0"},
                                     {"VQB_JIT_FACTOR": "1", "VQB_MIXED_SPLIT": "0"},
                                     {"VQB_JIT_FACTOR": "1", "VQB_JIT_RANKONE": "0"},
                                     {"VQB_JIT_FACTOR": "1", "VQB_JIT_PAIRFACTOR": "0"},
                                     {"VQB_JIT_FACTOR": "1", "VQB_JIT_DOTPLAN": "0"}])
def test_structure_classes_and_generator_variants(dev, ref, monkeypatch, variant):
    """Specialised kernels key on which matrix entries are exactly zero, real or
    imaginary (structure-aware emission): angles that make entries vanish
    (Rx(pi): zero real parts; Ry(pi): a zero diagonal; Rz(0): the identity)
    must compile their own kernels and still match the reference, forward and
    adjoint, in every generator variant (diagonal runs off, no accumulator
    budget, eager relayouts, serial host planning, no derivative generators,
    scalar factoring and cost-model fusion forced on at this size (they
    switch on by themselves at >= 2^22 amplitudes), partial-lane reductions,
    row-wise derivative contractions, unbatched slot reductions, unsplit
    superoperator steps, channel steps without the rank-one form or without
    per-state scalars)."""
    monkeypatch.setenv("VQB_JIT", "1")
    for k, v in variant.items():
        monkeypatch.setenv(k, v)
    n = 14
    for angle in (0.7, math.pi, 0.0):
        c = Circuit()
        for q in range(1, n + 1):
            c.push_back(standard_gate(GateKind.H, [q]))
        for layer in range(2):
            for q in range(1, n):
                c.push_back(standard_gate(GateKind.Cnot, [q, q + 1]))
                c.push_back(parametric_gate(GateKind.Rz, [q + 1], angle + 0.1 * layer, True))
                c.push_back(standard_gate(GateKind.Cnot, [q, q + 1]))
            for q in range(1, n + 1):
                c.push_back(parametric_gate(GateKind.Rx, [q], angle, True))
                c.push_back(parametric_gate(GateKind.Ry, [q], angle, True))
        s = dev.pure_state(n)
        dev.apply_circuit(c, s)
        r = ref.pure_state(n)
        ref.apply_circuit(c, r)
        assert np.max(np.abs(dev.download(s) - ref.download(r))) <= 1e-12
        op = sum_z(n)
        loss, g = dev.gradient_pure(op, c, dev.pure_state(n))
        rloss, rg = ref.gradient_pure(op, c, ref.pure_state(n))
        # the loss and some gradients vanish at these angles: relative to
        # max(|ref|, 1) (the observable's scale), i.e. 1e-10 absolute near zero
        assert abs(loss - rloss) <= RTOL * max(abs(rloss), 1.0)
        assert np.max(np.abs(g - rg)) <= RTOL * max(np.max(np.abs(rg)), 1.0)
    w = circuits.config3(n=6, layers=1)
    loss, g = dev.gradient_mixed(w.observable, w.circuit, dev.mixed_state(6))
    rloss, rg = ref.gradient_mixed(w.observable, w.circuit, ref.mixed_state(6))
    assert abs(loss - rloss) <= RTOL * abs(rloss) and rel_err(g, rg) <= RTOL


@pytest.mark.parametrize("factor", ["0", "1"])
def test_mixed_gradient_channel_forms(dev, ref, monkeypatch, factor):
    """Channel steps of the density-matrix adjoint in every form the lowering
    picks: depolarizing (rank-one, c (1 + e J)), amplitude and phase damping
    (real scalar only), a Generic two-Kraus channel, a 2-qubit parametric gate
    (fSim: ket and bra half steps on two bits each, five shared gradient
    entries) and tied single-qubit rotations, against the reference's
    gradient_mixed (autodiff.hpp:184-329)."""
    from paper_2406_19212_b200.abi import ChannelKind, make_channel, standard_channel
    monkeypatch.setenv("VQB_JIT", "1")
    monkeypatch.setenv("VQB_JIT_FACTOR", factor)
    n = 7
    c = Circuit()
    for q in range(1, n + 1):
        c.push_back(standard_gate(GateKind.H, [q]))
        c.push_back(parametric_gate(GateKind.Ry, [q], 0.3 + 0.1 * q, True))
        c.push_back(standard_channel(ChannelKind.Depolarizing, q, 0.02))
        c.push_back(parametric_gate(GateKind.Rz, [q], -0.2 + 0.05 * q, True))
        c.push_back(standard_channel(ChannelKind.PhaseDamping, q, 0.03))
    for q in range(1, n):
        c.push_back(parametric_gate(GateKind.Fsim, [q, q + 1], [0.4, -0.3, 0.2, 0.7, -0.5], [True] * 5))
        c.push_back(standard_channel(ChannelKind.AmplitudeDamping, q, 0.05))
    g = 0.1
    k0 = np.array([[1, 0], [0, math.sqrt(1 - g)]], dtype=complex)
    k1 = np.array([[0, math.sqrt(g) * 0.6], [0, 0.8j * math.sqrt(g)]], dtype=complex)
    c.push_back(make_channel([3], [k0, k1]))
    for q in range(1, n + 1):
        c.push_back(parametric_gate(GateKind.Rx, [q], 0.15 * q, True))
    op = sum_z(n)
    loss, gr = dev.gradient_mixed(op, c, dev.mixed_state(n))
    rloss, rg = ref.gradient_mixed(op, c, ref.mixed_state(n))
    assert abs(loss - rloss) <= RTOL * abs(rloss)
    assert rel_err(gr, rg) <= RTOL
