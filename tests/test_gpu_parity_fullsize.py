"""GPU parity on the path the product actually runs, against the reference.

The specialised (NVRTC-generated) stage kernels switch on by themselves at
>= 2^20 amplitudes, and the density-matrix adjoint then uses the 16-register
geometry with in-register superoperators; nothing here overrides VQB_JIT, so
these tests exercise the default executor at its production tile programs
(17-22 bits above the tile). Checks:

* live against the unmodified reference (oracle/_ref/libvqcs_ref.so) on all
  host cores: config-1 family at 24 qubits and full config 1 at 28 qubits
  (whole final state, max-abs <= 1e-12; apply_circuit circuit.hpp:110-129),
  config-2 family at 22 and 24 qubits (loss, 600 per-gate and 16 tied
  gradients, gradient_pure autodiff.hpp:95-156), config-3 family at 10 and 11
  qubits (4^10, 4^11 entries; gradient_mixed autodiff.hpp:184-329), and a
  permutation-only circuit (X / CNOT / SWAP / Toffoli / Fredkin) at 24 qubits,
  bit-exact (np.array_equal) through the fused executor;
* against the reference's own outputs at BASELINE.json's full sizes, stored by
  tests/golden/make_fullsize_golden.py (run once on the GPU box host):
  config 2 (30 qubits) loss and gradients, config 3 (15-qubit density matrix)
  loss and gradients, config 1 (28q) and config 4 (33q, 128 GiB) through an
  amplitude sample and overlaps with seeded product states
  (tests/helpers.product_projections_*), which move by O(1) under a qubit
  relabelling or a transposed matrix.

Tolerances (BASELINE.json north_star): amplitudes max-abs 1e-12; expectation
values and gradients ||d||_inf / ||ref||_inf <= 1e-10; permutations bit-exact;
product projections (O(1) sums over 2^n terms) |d| <= 1e-9.
"""
import json
import os

import numpy as np
import pytest

from paper_2406_19212_b200 import circuits
from paper_2406_19212_b200.abi import Circuit, GateKind, standard_gate

from helpers import (product_projections_device, random_state, rel_err, sample_amplitudes,
                     sample_indices, state_projections)

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "fullsize.json")


@pytest.fixture(scope="module")
def fast_ref():
    import oracle
    if not oracle.reference_available():
        pytest.skip("oracle/_ref/libvqcs_ref.so not built")
    eng = oracle.reference()
    oracle.set_reference_threads(os.cpu_count() or 1)
    return eng


@pytest.fixture(scope="module")
def golden():
    if not os.path.exists(GOLDEN):
        pytest.skip("tests/golden/fullsize.json not generated")
    with open(GOLDEN) as f:
        return json.load(f)


def kernels_of(dev, fn):
    dev.profile_begin()
    fn()
    return dev.profile_end()


def c(z):
    return np.array([complex(a, b) for a, b in z])


# ---------------------------------------------------------------- live vs the reference
@pytest.mark.parametrize("rows,cols,cycles", [(4, 6, 20), (4, 7, 20)])
def test_random_circuit_whole_state_default_path(dev, fast_ref, rows, cols, cycles):
    """Config-1 family (24 qubits) and full config 1 (28 qubits, 785 gates)."""
    w = circuits.config1(rows=rows, cols=cols, cycles=cycles)
    n = w.num_qubits
    s = dev.pure_state(n)
    prof = kernels_of(dev, lambda: dev.apply_circuit(w.circuit, s))
    assert "k_regstage_jit" in prof, prof  # the default executor at this size
    got = dev.download(s)
    s.free()
    r = fast_ref.pure_state(n)
    fast_ref.apply_circuit(w.circuit, r)
    want = fast_ref.download(r)
    r.free()
    err = float(np.max(np.abs(got - want)))
    assert err <= 1e-12, err
    assert abs(np.vdot(got, got).real - 1) <= 1e-11


@pytest.mark.parametrize("n", [22, 24])
def test_qaoa_gradient_default_path(dev, fast_ref, n):
    """Config-2 family: loss, 600 per-gate and 16 tied gradients."""
    w = circuits.config2(n=n)
    s0 = dev.pure_state(n)
    out = {}
    prof = kernels_of(dev, lambda: out.update(zip(("loss", "g"), dev.gradient_pure(w.observable, w.circuit, s0))))
    assert "k_regstage_rev_jit" in prof, prof
    r0 = fast_ref.pure_state(n)
    rl, rg = fast_ref.gradient_pure(w.observable, w.circuit, r0)
    assert abs(out["loss"] - rl) <= 1e-10 * max(abs(rl), 1e-300)
    assert len(out["g"]) == len(rg) == 20 * n  # p (|E| + n) = 8 (3n/2 + n)
    assert rel_err(out["g"], rg) <= 1e-10
    p, ne = w.extra["p"], len(w.extra["edges"])
    assert rel_err(circuits.qaoa_tied_gradients(out["g"], n, ne, p),
                   circuits.qaoa_tied_gradients(rg, n, ne, p)) <= 1e-10


@pytest.mark.parametrize("n", [10, 11])
def test_noisy_gradient_default_path(dev, fast_ref, n):
    """Config-3 family on 4^10 / 4^11 entries: the 16-register adjoint with
    in-register 2-qubit-channel superoperators."""
    w = circuits.config3(n=n)
    d0 = dev.mixed_state(n)
    out = {}
    prof = kernels_of(dev, lambda: out.update(zip(("loss", "g"), dev.gradient_mixed(w.observable, w.circuit, d0))))
    assert "k_regstage_rev_jit" in prof, prof
    r0 = fast_ref.mixed_state(n)
    rl, rg = fast_ref.gradient_mixed(w.observable, w.circuit, r0)
    assert abs(out["loss"] - rl) <= 1e-10 * max(abs(rl), 1e-300)
    assert len(out["g"]) == len(rg)
    assert rel_err(out["g"], rg) <= 1e-10


def test_noisy_forward_density_matrix_default_path(dev, fast_ref):
    w = circuits.config3(n=11)
    d = dev.mixed_state(11)
    dev.apply_circuit(w.circuit, d)
    r = fast_ref.mixed_state(11)
    fast_ref.apply_circuit(w.circuit, r)
    err = float(np.max(np.abs(dev.download(d) - fast_ref.download(r))))
    assert err <= 1e-12, err


def test_permutation_circuit_bit_exact(dev, fast_ref):
    """X / CNOT / SWAP / Toffoli / Fredkin only: every output amplitude is an
    input amplitude moved, so the fused executor must reproduce the reference
    bit for bit (kernels.hpp:291-299 moves data; fused 0/1 matrices must too)."""
    n = 24
    rng = np.random.default_rng(11)
    gates = []
    for _ in range(400):
        k = int(rng.integers(5))
        q = [int(x) + 1 for x in rng.choice(n, size=3, replace=False)]
        kind = [GateKind.X, GateKind.Cnot, GateKind.Swap, GateKind.Toffoli, GateKind.Fredkin][k]
        gates.append(standard_gate(kind, q[:[1, 2, 2, 3, 3][k]]))
    c = Circuit(gates)
    psi = random_state(n, rng)
    s = dev.from_amplitudes(psi)
    dev.apply_circuit(c, s)
    r = fast_ref.from_amplitudes(psi)
    fast_ref.apply_circuit(c, r)
    assert np.array_equal(dev.download(s), fast_ref.download(r))


# ---------------------------------------------------------------- the reference's full-size outputs
def test_config2_full_size_vs_reference(dev, golden):
    g = golden.get("config2") or pytest.skip("config2 not in fullsize.json")
    w = circuits.config2()
    loss, grads = dev.gradient_pure(w.observable, w.circuit, dev.pure_state(w.num_qubits))
    assert abs(loss - g["loss"]) <= 1e-10 * abs(g["loss"])
    assert rel_err(grads, np.array(g["grads"])) <= 1e-10
    tied = circuits.qaoa_tied_gradients(grads, w.num_qubits, len(w.extra["edges"]), w.extra["p"])
    assert rel_err(tied, np.array(g["tied"])) <= 1e-10
    dev.release_caches()


def test_config3_full_size_vs_reference(dev, golden):
    g = golden.get("config3") or pytest.skip("config3 not in fullsize.json")
    w = circuits.config3()
    loss, grads = dev.gradient_mixed(w.observable, w.circuit, dev.mixed_state(w.num_qubits))
    assert abs(loss - g["loss"]) <= 1e-10 * abs(g["loss"])
    assert rel_err(grads, np.array(g["grads"])) <= 1e-10
    dev.release_caches()


@pytest.mark.parametrize("name", ["config1", "config4"])
def test_random_circuit_full_size_vs_reference(dev, golden, name):
    g = golden.get(name) or pytest.skip(f"{name} not in fullsize.json")
    w = circuits.config1() if name == "config1" else circuits.config4(num_gpus=1)
    n = w.num_qubits
    assert n == g["n"] and len(w.circuit) == g["elements"]
    s = dev.pure_state(n)
    dev.apply_circuit(w.circuit, s)
    assert abs(dev.norm(s) - g["norm"]) <= 1e-11
    idx = np.array(g["sample_index"], dtype=np.int64)
    assert np.array_equal(idx, sample_indices(n))
    err = float(np.max(np.abs(sample_amplitudes(dev, s, idx) - c(g["sample"]))))
    assert err <= 1e-12, err
    if "product_projections" in g:
        pp = product_projections_device(dev, s, n)
        perr = float(np.max(np.abs(pp - c(g["product_projections"]))))
        assert perr <= 1e-9, perr
    if "projections" in g and n <= 28:  # hashed-weight projections (host side, chunked)
        hp = state_projections(dev, s, 1 << n)
        herr = float(np.max(np.abs(hp - c(g["projections"]))))
        assert herr <= 1e-9, herr
    s.free()
