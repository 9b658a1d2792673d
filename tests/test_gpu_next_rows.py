"""GPU: SURVEY §8(f) rows on the device — measure (circuit.hpp:303-375),
state dumps (io.hpp:40-128) and circuits rewritten by fuse_gates
(circuit.hpp:199-276) — against the reference (oracle/_ref) or the pinned
restatement."""
import numpy as np
import pytest

import oracle
from paper_2406_19212_b200 import circuits
from paper_2406_19212_b200.abi import IndexError_, IoError, TypeError_

from helpers import random_density, random_state

pytestmark = pytest.mark.gpu
needs_ref = pytest.mark.skipif(not oracle.reference_available(), reason="oracle/_ref not built")


def measure_ref(ref, amps, mixed, q, seed):
    """Outcome, probability and collapsed state of the reference's measure()
    on std::mt19937_64(seed)."""
    s = ref.from_amplitudes(amps, mixed)
    o, p = oracle.reference_measure(s, q, seed)
    return o, p, ref.download(s)


@needs_ref
@pytest.mark.parametrize("mixed", [False, True])
def test_measure_matches_reference(dev, ref, mixed):
    rng = np.random.default_rng(21 + mixed)
    for trial in range(12):
        n = int(rng.integers(2, 8 if mixed else 21))
        amps = random_density(n, rng) if mixed else random_state(n, rng)
        q = int(rng.integers(1, n + 1))
        seed = int(rng.integers(0, 2**63))
        o_ref, p_ref, after = measure_ref(ref, amps, mixed, q, seed)
        s = dev.from_amplitudes(amps, mixed)
        o, p = dev.measure(s, q, oracle.reference_uniform(seed))
        assert o == o_ref
        assert abs(p - p_ref) <= 1e-12 * max(p_ref, 1e-300)
        assert np.max(np.abs(dev.download(s) - after)) <= 1e-12


@needs_ref
def test_measure_halves_for_sharded_callers(dev, ref):
    rng = np.random.default_rng(4)
    amps = random_state(12, rng)
    s = dev.from_amplitudes(amps)
    p1 = dev.measure_probability(s, 5)
    want = float(np.sum(np.abs(amps[(np.arange(amps.size) >> 4) & 1 == 1]) ** 2))
    assert abs(p1 - want) <= 1e-13
    dev.collapse(s, 5, 0, 1.0 - p1)
    out = dev.download(s)
    assert np.all(out[(np.arange(amps.size) >> 4) & 1 == 1] == 0)
    assert abs(np.linalg.norm(out) - 1.0) <= 1e-12
    with pytest.raises(IndexError_):
        dev.measure(s, 13, 0.5)


@needs_ref
@pytest.mark.parametrize("n", [9, 23])  # 23 qubits = 128 MiB: two pinned chunks
def test_state_dump_byte_identical_and_loadable(dev, ref, tmp_path, n):
    rng = np.random.default_rng(n)
    amps = random_state(n, rng)
    pd, pr = tmp_path / "dev.vqcs", tmp_path / "ref.vqcs"
    dev.save_state(dev.from_amplitudes(amps), pd)
    ref.save_state(ref.from_amplitudes(amps), pr)
    assert pd.read_bytes() == pr.read_bytes()
    s, prec = dev.load_state(pr)
    assert prec == 2 and s.n == n
    assert np.array_equal(dev.download(s), amps)


@needs_ref
def test_state_dump_errors(dev, tmp_path):
    with pytest.raises(TypeError_):
        dev.save_state(dev.mixed_state(2), tmp_path / "dm.vqcs")
    with pytest.raises(IoError):
        dev.load_state(tmp_path / "absent.vqcs")
    bad = tmp_path / "short.vqcs"
    bad.write_bytes(b"VQCS" + (1).to_bytes(4, "little") + (3).to_bytes(4, "little") + b"\x02" + bytes(16))
    with pytest.raises(IoError):
        dev.load_state(bad)


def test_fused_circuit_on_device(dev, ref):
    c = circuits.config1(3, 4, 8).circuit
    s = dev.pure_state(12)
    dev.apply_circuit(dev.fuse_gates(c), s)
    r = ref.pure_state(12)
    ref.apply_circuit(c, r)
    assert np.max(np.abs(dev.download(s) - ref.download(r))) <= 1e-12
