"""GPU: API contracts beyond numerics.

* memory contract of the gradient sweep (tests/test_autodiff.cpp:132-145 in
  the reference: "only two working states live during the reverse sweep"),
  via vqb_alloc_stats (state_alloc_stats, state.hpp:154-161), and
  vqb_release_caches returning every cached working state;
* vqb_reverse_sweep accumulates into grads[grad_index + p] (+=), also when
  steps share an index (tied parameters), like the reference loop;
* bitwise run-to-run determinism of the reductions and gradients (fixed
  grids, fixed-order block sums; the reference's analogue is
  tests/test_kernels.cpp:209-230, identical results across thread counts);
* states on a non-zero current device (the adjoint worker thread
  must follow the caller's device) when a second GPU exists.
"""
import numpy as np
import pytest

from paper_2406_19212_b200 import circuits
from paper_2406_19212_b200.abi import GateKind, parametric_gate

from helpers import random_state, rel_err

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [12, 21])
def test_gradient_holds_two_working_states(dev, n):
    w = circuits.config0(n=n, layers=2)
    s0 = dev.pure_state(n)
    dev.release_caches()
    before = dev.alloc_stats()
    dev.reset_alloc_peak()
    dev.gradient_pure(w.observable, w.circuit, s0)
    during = dev.alloc_stats()
    assert during["peak"] - before["live"] <= 2, (before, during)  # Phi and Psi, nothing else
    dev.release_caches()
    after = dev.alloc_stats()
    assert after["live"] == before["live"], (before, after)
    assert after["live_bytes"] <= before["live_bytes"]
    s0.free()
    assert dev.alloc_stats()["live"] == before["live"] - 1


def test_reverse_sweep_accumulates_tied_indices(dev, ref):
    n = 10
    rng = np.random.default_rng(4)
    phi0, psi0 = random_state(n, rng), random_state(n, rng)
    steps = []
    for k in range(6):
        g = parametric_gate(GateKind.Ry, [1 + k % n], float(rng.uniform(-2, 2)), True)
        # steps 0, 2, 4 share slot 0; 1, 3, 5 share slot 1
        steps.append(([1 + k % n], ref.gate_inverse(g), [ref.gate_derivative(g, 0)], k % 2))
    out = {}
    for name, eng in (("dev", dev), ("ref", ref)):
        a, b = eng.from_amplitudes(phi0), eng.from_amplitudes(psi0)
        grads = np.full(2, 0.25)  # += semantics: the initial values stay
        eng.reverse_sweep(a, b, steps, 2.0, grads)
        out[name] = grads
    assert rel_err(out["dev"] - 0.25, out["ref"] - 0.25) <= 1e-12, out


def test_bitwise_run_to_run(dev):
    w = circuits.config2(n=22, p=2)
    s0 = dev.pure_state(22)
    l1, g1 = dev.gradient_pure(w.observable, w.circuit, s0)
    l2, g2 = dev.gradient_pure(w.observable, w.circuit, s0)
    assert l1 == l2 and np.array_equal(g1, g2)
    c = circuits.config1(rows=2, cols=11, cycles=8).circuit
    outs = []
    for _ in range(2):
        s = dev.pure_state(22)
        dev.apply_circuit(c, s)
        outs.append((dev.download(s), dev.norm(s), dev.expectation(w.observable, s)))
    assert np.array_equal(outs[0][0], outs[1][0])
    assert outs[0][1] == outs[1][1] and outs[0][2] == outs[1][2]
    d = circuits.config3(n=10, layers=2)
    r1 = dev.gradient_mixed(d.observable, d.circuit, dev.mixed_state(10))
    r2 = dev.gradient_mixed(d.observable, d.circuit, dev.mixed_state(10))
    assert r1[0] == r2[0] and np.array_equal(r1[1], r2[1])


def test_second_device_gradient(dev, ref):
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("one GPU on this box")
    torch.cuda.set_device(1)
    try:
        w = circuits.config0(n=12, layers=2)
        loss, g = dev.gradient_pure(w.observable, w.circuit, dev.pure_state(12))
        rl, rg = ref.gradient_pure(w.observable, w.circuit, ref.pure_state(12))
        assert abs(loss - rl) <= 1e-10 and rel_err(g, rg) <= 1e-10
    finally:
        torch.cuda.set_device(0)


@pytest.mark.parametrize("variant", [{}, {"VQB_JIT_FACTOR": "1"}, {"VQB_REV_REGS": "16"}])
def test_bounds_checked_kernels(dev, ref, monkeypatch, variant):
    """VQB_JIT_CHECK=1 compiles every specialised kernel with bounds checks on
    each global, shared-memory-tile and matrix-pool index (a violation traps
    and the call fails); with them on, forward, adjoint and density-matrix
    programs still match the reference. (compute-sanitizer is not allowed on
    this pool; this is the library's own check.)"""
    monkeypatch.setenv("VQB_JIT", "1")
    monkeypatch.setenv("VQB_JIT_CHECK", "1")
    for k, v in variant.items():
        monkeypatch.setenv(k, v)
    w = circuits.config1(rows=3, cols=5, cycles=8)
    s = dev.pure_state(15)
    dev.apply_circuit(w.circuit, s)
    r = ref.pure_state(15)
    ref.apply_circuit(w.circuit, r)
    assert np.max(np.abs(dev.download(s) - ref.download(r))) <= 1e-12
    for q in (circuits.config2(n=14, p=2), circuits.config0(n=13, layers=2)):
        loss, g = dev.gradient_pure(q.observable, q.circuit, dev.pure_state(q.num_qubits))
        rl, rg = ref.gradient_pure(q.observable, q.circuit, ref.pure_state(q.num_qubits))
        assert abs(loss - rl) <= 1e-10 * max(1.0, abs(rl)) and rel_err(g, rg) <= 1e-10
    d = circuits.config3(n=6, layers=2)
    loss, g = dev.gradient_mixed(d.observable, d.circuit, dev.mixed_state(6))
    rl, rg = ref.gradient_mixed(d.observable, d.circuit, ref.mixed_state(6))
    assert abs(loss - rl) <= 1e-10 * max(1.0, abs(rl)) and rel_err(g, rg) <= 1e-10


def test_async_upload_from_pinned_memory(dev):
    """vqb_state_upload_async: ordered on the state's stream (the following
    gradient sees the uploaded state), pageable memory is refused."""
    import torch
    from paper_2406_19212_b200.abi import UsageError
    n = 14
    w = circuits.config0(n=n, layers=2)
    rng = np.random.default_rng(5)
    amps = random_state(n, rng)
    s_sync = dev.pure_state(n)
    dev.upload(s_sync, amps)
    want = dev.gradient_pure(w.observable, w.circuit, s_sync)
    pinned = torch.zeros(2 << n, dtype=torch.float64, pin_memory=True)
    pinned.numpy().view(np.complex128)[:] = amps
    s = dev.pure_state(n)
    dev.upload_async(s, pinned.data_ptr(), 1 << n)
    got = dev.gradient_pure(w.observable, w.circuit, s)
    assert got[0] == want[0] and np.array_equal(got[1], want[1])
    pageable = np.ascontiguousarray(amps)
    with pytest.raises(UsageError):
        dev.upload_async(s, pageable.ctypes.data, 1 << n)
    s.free()
    s_sync.free()
