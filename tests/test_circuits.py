"""CPU: the seeded generators (paper_2406_19212_b200.circuits) — RNG restated
from rng.hpp:31-71, config shapes from BASELINE.json / SURVEY.md §8(d)."""
import math

import numpy as np

from paper_2406_19212_b200 import circuits
from paper_2406_19212_b200.abi import ChannelOp, GateKind, GateOp


def test_splitmix64_known_values():
    # SplitMix64(0) first outputs (Steele et al.; rng.hpp:38-49)
    r = circuits.SplitMix64(0)
    assert [r.next() for _ in range(3)] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4,
                                            0x06C45D188009454F]
    u = circuits.SplitMix64(1).next_unit()
    assert 0 < u <= 1


def test_child_stream_is_order_independent():
    a = circuits.child_stream(7, 3, 5).next()
    circuits.child_stream(7, 2, 5).next()
    assert circuits.child_stream(7, 3, 5).next() == a
    assert circuits.child_stream(7, 3, 6).next() != a


def test_config_shapes():
    w0 = circuits.config0()
    assert len(w0.circuit) == 790 and w0.circuit.num_active_params() == 600
    w1 = circuits.config1()
    kinds = [e.kind for e in w1.circuit.elements]
    assert len(kinds) == 785 and kinds.count(GateKind.Fsim) == 225
    assert sum(1 for e in w1.circuit.elements if e.kind == GateKind.Generic) > 100  # sqrt(W)
    # never the same 1q gate twice in a row on a qubit
    last = {}
    for e in w1.circuit.elements:
        if len(e.positions) == 1:
            key = (e.kind, None if e.matrix is None else e.matrix.tobytes())
            assert last.get(e.positions[0]) != key
            last[e.positions[0]] = key
    w2 = circuits.config2()
    assert len(w2.extra["edges"]) == 45
    deg = np.zeros(31, int)
    for i, j in w2.extra["edges"]:
        deg[i] += 1
        deg[j] += 1
    assert (deg[1:] == 3).all()
    assert w2.circuit.num_active_params() == 8 * (45 + 30)
    w3 = circuits.config3()
    assert len(w3.circuit) == 798 and w3.circuit.num_active_params() == 270
    assert sum(isinstance(e, ChannelOp) for e in w3.circuit.elements) == 6 * (45 + 14 + 15)
    for g, (rows, cols) in circuits.CONFIG4_GRIDS.items():
        w4 = circuits.config4(g)
        assert w4.num_qubits == rows * cols


def test_sqrt_w_is_a_square_root_of_w():
    w = (np.array([[0, 1], [1, 0]]) + np.array([[0, -1j], [1j, 0]])) / math.sqrt(2)
    s = circuits.SQRT_W
    assert np.allclose(s.conj().T @ s, np.eye(2), atol=1e-15)
    assert np.allclose(s @ s, w, atol=1e-15)  # the pinned convention: sqrt(W)^2 = W exactly


def test_depolarizing2_is_complete():
    k = circuits.depolarizing2_kraus(0.01)
    s = sum(x.conj().T @ x for x in k)
    assert np.allclose(s, np.eye(4), atol=1e-15) and len(k) == 16


def test_tied_gradient_chain_rule():
    g = np.arange(2 * (3 + 4), dtype=float)
    t = circuits.qaoa_tied_gradients(g, 4, 3, 2)
    assert list(t) == [2 * (0 + 1 + 2), 2 * (7 + 8 + 9), 2 * (3 + 4 + 5 + 6), 2 * (10 + 11 + 12 + 13)]
