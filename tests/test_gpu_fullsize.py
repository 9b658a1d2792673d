"""GPU, BASELINE.json's full sizes, through size-independent properties (the
CPU oracle cannot run these sizes in test time):

* config 4 at 33 qubits (128 GiB) and config 1 at 28 qubits: the circuit
  preserves the norm, and the circuit followed by its inverse (the
  reference's gate_inverse, gates.hpp:581-619, in reverse order) returns
  |0...0> (a round trip);
* config 2 (30 qubits) and config 3 (15-qubit density matrix, 2^30 entries):
  adjoint gradients agree with central finite differences of the device loss
  on sampled parameters; the density matrix keeps unit trace.

Tolerances: round trip / norm 1e-11 (785-1500 gate applications at ~1e-16
each); finite differences h = 1e-4: truncation ~h^2 * |g'''|, rounding
~1e-16 / h, so |g - fd| <= 1e-6 * max(1, |g|)."""
import math

import numpy as np
import pytest

from paper_2406_19212_b200 import circuits
from paper_2406_19212_b200.abi import Circuit, GateOp, make_gate, sum_z

pytestmark = pytest.mark.gpu


def inverse_circuit(dev, c):
    return Circuit([make_gate(list(e.positions), dev.gate_inverse(e).reshape(-1))
                    for e in reversed(c.elements)])


def perturbed(c, p, h):
    """Copy of circuit c with its p-th active parameter (traversal order,
    circuit.hpp:149-159) shifted by h."""
    out, k = [], 0
    for e in c.elements:
        if isinstance(e, GateOp) and e.num_active_params():
            params = list(e.params)
            for j, act in enumerate(e.is_param):
                if act:
                    if k == p:
                        params[j] += h
                    k += 1
            e = GateOp(list(e.positions), e.kind, params, list(e.is_param), e.matrix)
        out.append(e)
    return Circuit(out)


def test_config4_33_qubits_norm_and_round_trip(dev):
    w = circuits.config4(num_gpus=1)
    s = dev.pure_state(w.num_qubits)
    dev.apply_circuit(w.circuit, s)
    assert abs(dev.norm(s) - 1.0) <= 1e-11
    dev.apply_circuit(inverse_circuit(dev, w.circuit), s)
    # back on |0...0>: every <Z_q> = 1 (the state is too large to download)
    assert abs(dev.norm(s) - 1.0) <= 1e-11
    assert abs(dev.expectation(sum_z(w.num_qubits), s).real - w.num_qubits) <= 1e-10
    s.free()


def test_config1_round_trip_is_exact_to_rounding(dev):
    w = circuits.config1()
    s = dev.pure_state(28)
    dev.apply_circuit(w.circuit, s)
    assert abs(dev.norm(s) - 1.0) <= 1e-12
    dev.apply_circuit(inverse_circuit(dev, w.circuit), s)
    a = dev.download(s)
    assert abs(a[0] - 1.0) <= 1e-11
    assert np.max(np.abs(a[1:])) <= 1e-11
    s.free()


def check_fd(dev, w, mixed, params):
    s0 = dev.mixed_state(w.num_qubits) if mixed else dev.pure_state(w.num_qubits)
    grad = dev.gradient_mixed if mixed else dev.gradient_pure
    loss_fn = dev.loss_mixed if mixed else dev.loss_pure
    loss, g = grad(w.observable, w.circuit, s0)
    assert abs(loss_fn(w.observable, w.circuit, s0) - loss) <= 1e-10 * max(1.0, abs(loss))
    h = 1e-4
    for p in params:
        up = loss_fn(w.observable, perturbed(w.circuit, p, h), s0)
        dn = loss_fn(w.observable, perturbed(w.circuit, p, -h), s0)
        fd = (up - dn) / (2 * h)
        assert abs(g[p] - fd) <= 1e-6 * max(1.0, abs(g[p])), (p, g[p], fd)
    s0.free()
    return g


def test_config2_30_qubit_gradient_vs_finite_differences(dev):
    w = circuits.config2()
    g = check_fd(dev, w, False, [0, 44, 45 + 7, 599])
    assert g.shape == (600,)


def test_config3_noisy_gradient_vs_finite_differences_and_trace(dev):
    w = circuits.config3()
    s = dev.mixed_state(w.num_qubits)
    dev.apply_circuit(w.circuit, s)
    assert abs(dev.trace(s) - 1.0) <= 1e-12
    s.free()
    g = check_fd(dev, w, True, [0, 1, 134, 269])
    assert g.shape == (270,)
