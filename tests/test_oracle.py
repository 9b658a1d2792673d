"""CPU: pin the oracle (test infrastructure) before trusting it.

* the plain-C restatement (oracle/vqcs_oracle.c) against the reference itself
  (oracle/_ref/libvqcs_ref.so, compiled from /root/reference);
* both against the golden vectors generated from the reference
  (tests/golden/make_golden.py) and the reference tests' known answers
  (tests/test_kernels.cpp, test_autodiff.cpp, test_observables.cpp).
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
from paper_2406_19212_b200 import circuits
from paper_2406_19212_b200.abi import (ChannelKind, Circuit, GateKind, NonInvertibleChannelError,
                                       PauliOperator, PauliTerm, heisenberg_1d, make_gate,
                                       parametric_gate, standard_channel, standard_gate)

from helpers import (random_channel, random_density, random_gate, random_operator, random_state,
                     rel_err)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
needs_ref = pytest.mark.skipif(not oracle.reference_available(), reason="oracle/_ref not built")


@pytest.fixture(scope="module")
def golden():
    with open(os.path.join(GOLDEN, "golden.json")) as f:
        return json.load(f)


def z_on(q):
    return PauliOperator([PauliTerm([(q, "z")], 1.0)])


def test_known_answers_restatement(orc):
    s = orc.pure_state(1)
    orc.apply_gate(s, standard_gate(GateKind.H, [1]))
    assert np.allclose(orc.download(s), [2 ** -0.5] * 2, atol=1e-15)
    assert orc.expectation(heisenberg_1d(3), orc.pure_state(3)).real == pytest.approx(5.0)
    for theta in (0.0, 0.3, math.pi / 2, 1.9):
        c = Circuit([parametric_gate(GateKind.Rx, [1], theta, True)])
        loss, g = orc.gradient_pure(z_on(1), c, orc.pure_state(1))
        assert loss == pytest.approx(math.cos(theta), abs=1e-12)
        assert g[0] == pytest.approx(-math.sin(theta), abs=1e-10)
    p = 0.3
    c = Circuit([parametric_gate(GateKind.Rx, [1], 0.7, True),
                 standard_channel(ChannelKind.Depolarizing, 1, p)])
    loss, g = orc.gradient_mixed(z_on(1), c, orc.mixed_state(1))
    assert loss == pytest.approx((1 - p) * math.cos(0.7), abs=1e-10)
    assert g[0] == pytest.approx(-(1 - p) * math.sin(0.7), abs=1e-9)
    c = Circuit([parametric_gate(GateKind.Rx, [1], 0.4, True),
                 standard_channel(ChannelKind.AmplitudeDamping, 1, 1.0)])
    with pytest.raises(NonInvertibleChannelError):
        orc.gradient_mixed(z_on(1), c, orc.mixed_state(1))


def test_golden_config0_restatement(orc, golden):
    g0 = golden["config0"]
    w = circuits.config0()
    loss, g, res = orc.gradient_pure(w.observable, w.circuit, orc.pure_state(20), with_residual=True)
    assert abs(loss - g0["loss"]) <= 1e-10 * abs(g0["loss"])
    assert rel_err(g, g0["grads"]) <= 1e-10
    assert res <= 1e-8
    # SURVEY.md §8(c) values computed independently at survey time
    assert loss == pytest.approx(0.19589280189123967, abs=1e-13)
    assert g[1] == pytest.approx(-0.18247336625452928, abs=1e-13)


def test_golden_small_configs_restatement(orc, golden):
    w = circuits.config1(rows=3, cols=4, cycles=8)
    s = orc.pure_state(12)
    orc.apply_circuit(w.circuit, s)
    want = np.load(os.path.join(GOLDEN, "config1_3x4_8cyc_state.npy"))
    assert np.max(np.abs(orc.download(s) - want)) <= 1e-13
    w = circuits.config2(n=10, p=3)
    loss, g = orc.gradient_pure(w.observable, w.circuit, orc.pure_state(10))
    gd = golden["config2_10_p3"]
    assert abs(loss - gd["loss"]) <= 1e-10 * abs(gd["loss"])
    assert rel_err(g, gd["grads"]) <= 1e-10
    assert [list(e) for e in w.extra["edges"]] == gd["edges"]
    w = circuits.config3(n=4, layers=2)
    loss, g = orc.gradient_mixed(w.observable, w.circuit, orc.mixed_state(4))
    gd = golden["config3_4_2l"]
    assert abs(loss - gd["loss"]) <= 1e-10 * abs(gd["loss"])
    assert rel_err(g, gd["grads"]) <= 1e-10
    dm = orc.mixed_state(4)
    orc.apply_circuit(w.circuit, dm)
    assert np.max(np.abs(orc.download(dm) - np.load(os.path.join(GOLDEN, "config3_4_2l_rho.npy")))) <= 1e-13


@needs_ref
def test_restatement_matches_reference_gates(orc):
    ref = oracle.reference()
    oracle.set_reference_threads(1)
    rng = np.random.default_rng(5)
    for _ in range(80):
        n = int(rng.integers(2, 10))
        g = random_gate(n, rng)
        amps = random_state(n, rng)
        a, b = orc.from_amplitudes(amps), ref.from_amplitudes(amps)
        orc.apply_gate(a, g)
        ref.apply_gate(b, g)
        # same operation order, no FMA contraction: bit-identical
        assert np.array_equal(orc.download(a), ref.download(b))
        assert np.array_equal(orc.gate_matrix(g), ref.gate_matrix(g))
        assert np.array_equal(orc.gate_inverse(g), ref.gate_inverse(g))


@needs_ref
def test_restatement_matches_reference_channels_and_observables(orc):
    ref = oracle.reference()
    rng = np.random.default_rng(6)
    for _ in range(10):
        n = 3
        elems = [random_channel(n, rng) if rng.integers(2) else random_gate(n, rng, max_targets=2)
                 for _ in range(10)]
        c = Circuit(elems)
        rho = random_density(n, rng)
        a, b = orc.from_amplitudes(rho, True), ref.from_amplitudes(rho, True)
        orc.apply_circuit(c, a)
        ref.apply_circuit(c, b)
        assert np.max(np.abs(orc.download(a) - ref.download(b))) <= 1e-14
        op = random_operator(n, 5, rng)
        assert abs(orc.expectation(op, a) - ref.expectation(op, b)) <= 1e-14
        for e in elems:
            if not isinstance(e, type(elems[0])) or True:
                pass
        ch = random_channel(n, rng)
        assert np.max(np.abs(orc.channel_superop(ch) - ref.channel_superop(ch))) <= 1e-15


@needs_ref
def test_restatement_matches_reference_gradients(orc):
    ref = oracle.reference()
    rng = np.random.default_rng(7)
    n = 6
    c = Circuit([random_gate(n, rng, active=True) for _ in range(40)])
    op = random_operator(n, 6, rng)
    l1, g1 = orc.gradient_pure(op, c, orc.pure_state(n))
    l2, g2 = ref.gradient_pure(op, c, ref.pure_state(n))
    assert abs(l1 - l2) <= 1e-12 and rel_err(g1, g2) <= 1e-12
    w = circuits.config3(n=3, layers=1)
    l1, g1 = orc.gradient_mixed(w.observable, w.circuit, orc.mixed_state(3))
    l2, g2 = ref.gradient_mixed(w.observable, w.circuit, ref.mixed_state(3))
    assert abs(l1 - l2) <= 1e-12 and rel_err(g1, g2) <= 1e-12


def test_finite_difference_consistency(orc):
    """Independent check of the restated adjoint: central differences
    (finite_difference_gradient autodiff.hpp:333-354, h = 1e-5)."""
    w = circuits.config0(n=4, layers=2)
    loss, g = orc.gradient_pure(w.observable, w.circuit, orc.pure_state(4))
    params = w.circuit.active_parameters()
    fd = []
    for j in range(len(params)):
        up, dn = list(params), list(params)
        up[j] += 1e-5
        dn[j] -= 1e-5
        w.circuit.reset_parameters(up)
        lu = orc.loss_pure(w.observable, w.circuit, orc.pure_state(4))
        w.circuit.reset_parameters(dn)
        ld = orc.loss_pure(w.observable, w.circuit, orc.pure_state(4))
        fd.append((lu - ld) / 2e-5)
    w.circuit.reset_parameters(params)
    assert np.max(np.abs(np.array(fd) - g)) <= 1e-6
