"""GPU: the CUDA path against the golden vectors generated from the reference
(tests/golden/make_golden.py), so parity is pinned even where /root/reference
is absent."""
import json
import os

import numpy as np
import pytest

from paper_2406_19212_b200 import circuits

from helpers import rel_err

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def golden():
    with open(os.path.join(GOLDEN, "golden.json")) as f:
        return json.load(f)


def test_config0_full_size(dev, golden):
    g0 = golden["config0"]
    w = circuits.config0()
    loss, g, res = dev.gradient_pure(w.observable, w.circuit, dev.pure_state(20), with_residual=True)
    assert abs(loss - g0["loss"]) <= 1e-10 * abs(g0["loss"])
    assert rel_err(g, g0["grads"]) <= 1e-10
    assert res <= 1e-8
    s = dev.pure_state(20)
    dev.apply_circuit(w.circuit, s)
    a0 = dev.download(s)[0]
    assert abs(a0 - complex(*g0["amp0"])) <= 1e-12


@pytest.mark.parametrize("fused", [True, False])
def test_config1_reduced_state(dev, fused):
    w = circuits.config1(rows=3, cols=4, cycles=8)
    s = dev.pure_state(12)
    dev.apply_circuit(w.circuit, s, fused=fused)
    want = np.load(os.path.join(GOLDEN, "config1_3x4_8cyc_state.npy"))
    assert np.max(np.abs(dev.download(s) - want)) <= 1e-12


def test_config2_reduced(dev, golden):
    gd = golden["config2_10_p3"]
    w = circuits.config2(n=10, p=3)
    loss, g = dev.gradient_pure(w.observable, w.circuit, dev.pure_state(10))
    assert abs(loss - gd["loss"]) <= 1e-10 * abs(gd["loss"])
    assert rel_err(g, gd["grads"]) <= 1e-10
    tied = circuits.qaoa_tied_gradients(g, 10, len(gd["edges"]), 3)
    assert rel_err(tied, gd["tied"]) <= 1e-10


def test_config3_reduced(dev, golden):
    gd = golden["config3_4_2l"]
    w = circuits.config3(n=4, layers=2)
    loss, g = dev.gradient_mixed(w.observable, w.circuit, dev.mixed_state(4))
    assert abs(loss - gd["loss"]) <= 1e-10 * abs(gd["loss"])
    assert rel_err(g, gd["grads"]) <= 1e-10
    dm = dev.mixed_state(4)
    dev.apply_circuit(w.circuit, dm)
    want = np.load(os.path.join(GOLDEN, "config3_4_2l_rho.npy"))
    assert np.max(np.abs(dev.download(dm) - want)) <= 1e-12
    assert abs(dev.trace(dm) - complex(*gd["trace"])) <= 1e-12
