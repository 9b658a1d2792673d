"""GPU: the sharded executor's device engine (vqb_state_wrap over a torch CUDA
shard, fused executor on the shard) at world size 1; the multi-rank exchange
logic is covered by tests/test_distributed.py (gloo, CPU)."""
import numpy as np
import pytest
import torch

from paper_2406_19212_b200 import circuits
from paper_2406_19212_b200.distributed import DeviceEngine, ShardedState

pytestmark = pytest.mark.gpu


class NoDist:
    pass


def test_device_shard_matches_reference(dev, ref):
    w = circuits.config1(rows=3, cols=5, cycles=10)
    n = w.num_qubits
    st = ShardedState(n, NoDist(), DeviceEngine(dev),
                      torch.zeros(1 << n, dtype=torch.complex128, device="cuda"), 0, 1)
    st.set_zero()
    st.apply_circuit(w.circuit)
    r = ref.pure_state(n)
    ref.apply_circuit(w.circuit, r)
    assert np.max(np.abs(st.gather() - ref.download(r))) <= 1e-12
    assert abs(st.norm() - 1) <= 1e-12
    op = circuits.sum_z(n)
    assert abs(st.expectation(op) - ref.expectation(op, r)) <= 1e-12


def test_device_shard_gradient_matches_reference(dev, ref):
    """Sharded adjoint plumbing on the device (vqb_reverse_sweep over wrapped
    shards, apply_operator into a second shard) at world size 1."""
    w = circuits.config2(n=12, p=2, seed=5)
    n = w.num_qubits
    st = ShardedState(n, NoDist(), DeviceEngine(dev),
                      torch.zeros(1 << n, dtype=torch.complex128, device="cuda"), 0, 1)
    st.set_zero()
    loss, grads = st.gradient_pure(w.observable, w.circuit)
    want_loss, want = ref.gradient_pure(w.observable, w.circuit, ref.pure_state(n))
    assert abs(loss - want_loss) <= 1e-10 * max(1.0, abs(want_loss))
    assert np.max(np.abs(grads - want)) <= 1e-10 * max(1.0, np.max(np.abs(want)))


def test_reverse_sweep_matches_reference(dev, ref):
    """vqb_reverse_sweep (batched reverse_sweep_step, kernels.hpp:659-697)
    against the reference's own reverse_sweep_step applied step by step."""
    from helpers import random_state, random_unitary
    rng = np.random.default_rng(9)
    n = 14
    steps = []
    nslots = 0
    for _ in range(40):
        m = int(rng.integers(1, 3))
        pos = [int(x) + 1 for x in rng.choice(n, size=m, replace=False)]
        d = 1 << m
        inv = random_unitary(d, rng).reshape(-1, order="F")
        nd = int(rng.integers(0, 3))
        dm = [(rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))).reshape(-1, order="F")
              for _ in range(nd)]
        steps.append((pos, inv, dm, nslots))
        nslots += nd
    a, b = random_state(n, rng), random_state(n, rng)
    g_dev = np.zeros(nslots)
    g_ref = np.zeros(nslots)
    pa, pb = dev.from_amplitudes(a), dev.from_amplitudes(b)
    dev.reverse_sweep(pa, pb, steps, 2.0, g_dev)
    ra, rb = ref.from_amplitudes(a), ref.from_amplitudes(b)
    ref.reverse_sweep(ra, rb, steps, 2.0, g_ref)
    assert np.max(np.abs(dev.download(pa) - ref.download(ra))) <= 1e-12
    assert np.max(np.abs(dev.download(pb) - ref.download(rb))) <= 1e-12
    assert np.max(np.abs(g_dev - g_ref)) <= 1e-10 * np.max(np.abs(g_ref))
