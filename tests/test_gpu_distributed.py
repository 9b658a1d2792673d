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
