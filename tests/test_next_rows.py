"""CPU: SURVEY §8(f) rows around the path — fuse_gates (circuit.hpp:199-276),
measure (circuit.hpp:303-375) and state dumps (io.hpp:40-128).

The restatement is pinned against the reference (seeded std::mt19937_64
draws for measure, byte-identical dump files), and the product's host-only
fuse_gates is compared with the reference's here (no device needed); the
device measure/dump paths are covered by tests/test_gpu_next_rows.py.
"""
import os

import numpy as np
import pytest

import oracle
from paper_2406_19212_b200 import circuits
from paper_2406_19212_b200.abi import (Circuit, GateKind, IoError, IndexError_, TypeError_, UnsupportedError,
                                       make_gate, parametric_gate, standard_channel,
                                       standard_gate, ChannelKind, make_channel)

from helpers import random_density, random_gate, random_state, random_unitary

needs_ref = pytest.mark.skipif(not oracle.reference_available(), reason="oracle/_ref not built")


def fuse_cases():
    rng = np.random.default_rng(11)
    cases = [circuits.config1(3, 4, 6).circuit, circuits.config0(6, 3).circuit]
    for _ in range(6):  # random mixes of 1q/2q/3q gates, incl. parametric ones
        c = Circuit()
        for _ in range(int(rng.integers(1, 40))):
            c.push_back(random_gate(5, rng))
        cases.append(c)
    c = Circuit()  # a 1q gate between two eligible 2q gates merges into the later one
    c.push_back(standard_gate(GateKind.Cnot, [1, 2]))
    c.push_back(standard_gate(GateKind.H, [2]))
    c.push_back(parametric_gate(GateKind.Rz, [1], 0.3, True))
    c.push_back(standard_gate(GateKind.CZ, [2, 3]))
    c.push_back(standard_gate(GateKind.T, [4]))  # no 2q neighbour: survives
    cases.append(c)
    return cases


def same_ops(a, b, tol):
    assert len(a.elements) == len(b.elements)
    for x, y in zip(a.elements, b.elements):
        assert list(x.positions) == list(y.positions)
        assert np.max(np.abs(np.asarray(x.matrix) - np.asarray(y.matrix))) <= tol


@needs_ref
def test_fuse_gates_restatement_and_product_match_reference(orc, dev):
    ref = oracle.reference()
    for c in fuse_cases():
        r = ref.fuse_gates(c)
        same_ops(orc.fuse_gates(c), r, 0.0)      # same operation order: bit-identical
        same_ops(dev.fuse_gates(c), r, 1e-15)    # product (host-only call, no GPU)
    for eng in (ref, orc, dev):
        c = Circuit()
        c.push_back(standard_gate(GateKind.H, [1]))
        c.push_back(standard_channel(ChannelKind.Depolarizing, 1, 0.1))
        with pytest.raises(UnsupportedError):
            eng.fuse_gates(c)


@needs_ref
def test_fused_circuit_preserves_the_state(orc):
    ref = oracle.reference()
    c = circuits.config1(3, 4, 6).circuit
    a, b = ref.pure_state(12), ref.pure_state(12)
    ref.apply_circuit(c, a)
    ref.apply_circuit(ref.fuse_gates(c), b)
    assert np.max(np.abs(ref.download(a) - ref.download(b))) <= 1e-12


@needs_ref
def test_measure_restatement_matches_reference_draws(orc):
    ref = oracle.reference()
    rng = np.random.default_rng(3)
    for trial in range(24):
        mixed = trial % 3 == 2
        n = int(rng.integers(1, 4 if mixed else 8))
        amps = random_density(n, rng) if mixed else random_state(n, rng)
        q = int(rng.integers(1, n + 1))
        seed, skip = int(rng.integers(0, 2**63)), int(rng.integers(0, 5))
        u = oracle.reference_uniform(seed, skip)
        a = ref.from_amplitudes(amps, mixed)
        b = orc.from_amplitudes(amps, mixed)
        o_ref, p_ref = oracle.reference_measure(a, q, seed, skip)
        o, p = orc.measure(b, q, u)
        assert o == o_ref and p == p_ref
        assert np.array_equal(orc.download(b), ref.download(a))
        # measuring again repeats the outcome with probability 1
        o2, p2 = orc.measure(b, q, u)
        assert o2 == o and abs(p2 - 1.0) <= 1e-12


def test_measure_errors(orc):
    s = orc.pure_state(3)
    for bad in (0, 4):
        with pytest.raises(IndexError_):
            orc.measure(s, bad, 0.5)
    # a zero vector is not degenerate for the reference's clamping rule:
    # p1 = 0, p0 = clamp(1 - 0) = 1, so outcome 0 "with probability 1"
    z = orc.from_amplitudes(np.zeros(8, dtype=np.complex128))
    assert orc.measure(z, 1, 0.5) == (0, 1.0)
    if oracle.reference_available():
        zr = oracle.reference().from_amplitudes(np.zeros(8, dtype=np.complex128))
        assert oracle.reference_measure(zr, 1, 1234) == (0, 1.0)


@needs_ref
def test_state_dumps_byte_identical(orc, tmp_path):
    ref = oracle.reference()
    rng = np.random.default_rng(8)
    amps = random_state(7, rng)
    pr, po = tmp_path / "ref.vqcs", tmp_path / "orc.vqcs"
    ref.save_state(ref.from_amplitudes(amps), pr)
    orc.save_state(orc.from_amplitudes(amps), po)
    assert pr.read_bytes() == po.read_bytes()
    assert pr.read_bytes()[:13] == b"VQCS" + (1).to_bytes(4, "little") + (7).to_bytes(4, "little") + b"\x02"
    for eng in (ref, orc):
        s, prec = eng.load_state(pr)
        assert prec == 2 and s.n == 7
        assert np.array_equal(eng.download(s), amps)


@needs_ref
@pytest.mark.parametrize("case", ["magic", "version", "qubits", "precision", "truncated", "missing"])
def test_state_load_errors(orc, tmp_path, case):
    ref = oracle.reference()
    good = b"VQCS" + (1).to_bytes(4, "little") + (2).to_bytes(4, "little") + b"\x02" + bytes(64)
    data = {"magic": b"XQCS" + good[4:],
            "version": good[:4] + (2).to_bytes(4, "little") + good[8:],
            "qubits": good[:8] + (41).to_bytes(4, "little") + good[12:],
            "precision": good[:12] + b"\x03" + good[13:],
            "truncated": good[:-8],
            "missing": None}[case]
    path = tmp_path / "bad.vqcs"
    if data is not None:
        path.write_bytes(data)
    for eng in (ref, orc):
        with pytest.raises(IoError):
            eng.load_state(path)


def test_state_save_rejects_density_matrix(orc, tmp_path):
    with pytest.raises(TypeError_):
        orc.save_state(orc.mixed_state(2), tmp_path / "dm.vqcs")


# ---- analytic channel inverses (row f4): named channels in closed form,
# Generic ones by elimination; the reference inverts every channel by LU
# (autodiff.hpp:263-276, linalg.hpp:140-200)
@pytest.mark.parametrize("kind", [ChannelKind.AmplitudeDamping, ChannelKind.PhaseDamping,
                                  ChannelKind.Depolarizing])
@pytest.mark.parametrize("param", [0.0, 1e-3, 0.3, 0.999, 1 - 1e-13, 1.0])
def test_named_channel_inverse_matches_reference_lu(kind, param):
    import paper_2406_19212_b200 as vqb
    import oracle
    if not oracle.reference_available():
        pytest.skip("reference not built")
    dev, ref = vqb.device(), oracle.reference()
    ch = standard_channel(kind, 2, param)
    inv, cond = dev.channel_inverse(ch)
    rinv, rcond = ref.channel_inverse(ch)
    assert (inv is None) == (rinv is None)
    # the NonInvertibleChannelError decision (condition limit 1e12, autodiff.hpp:51)
    assert (inv is None or cond > 1e12) == (rinv is None or rcond > 1e12)
    if inv is not None:
        assert cond == pytest.approx(rcond, rel=1e-9)
        assert np.max(np.abs(inv - rinv)) <= 1e-12 * max(1.0, np.max(np.abs(rinv)))


def test_generic_channel_inverse_matches_reference_lu():
    import paper_2406_19212_b200 as vqb
    import oracle
    from paper_2406_19212_b200 import circuits
    if not oracle.reference_available():
        pytest.skip("reference not built")
    dev, ref = vqb.device(), oracle.reference()
    rng = np.random.default_rng(8)
    chans = [make_channel([1, 3], circuits.depolarizing2_kraus(1e-2))]
    for _ in range(5):  # random 1-qubit Kraus pairs (generic)
        u = random_unitary(4, rng)
        k0, k1 = u[:2, :2], u[2:, :2]  # isometry columns -> completeness holds
        chans.append(make_channel([2], [k0.reshape(-1, order="F"), k1.reshape(-1, order="F")]))
    for ch in chans:
        inv, cond = dev.channel_inverse(ch)
        rinv, rcond = ref.channel_inverse(ch)
        assert (inv is None) == (rinv is None)
        if inv is not None:
            assert cond == pytest.approx(rcond, rel=1e-9)
            assert np.max(np.abs(inv - rinv)) <= 1e-10 * max(1.0, np.max(np.abs(rinv)))


# ---- BenchRecord reports (row f3): byte-identical to the reference harness's
# emit_report (src/bench.cpp:329-369), JSON and CSV
BENCH_RECORDS = [
    {"task": "rqc", "n": 28, "depth": 20, "threads": 1, "seconds": [0.07422, 0.0739, 0.0745],
     "params": {"seed": "0", "verify_norm": "0.999999999999", "device": "B200 \"sm_100a\""}},
    {"task": "rqc-grad", "n": 30, "depth": 8, "threads": 16, "seconds": [1.0, 2.5e-05, 123456789.125, 1e-7],
     "params": {}},
    {"task": "thread-sweep", "n": 22, "depth": 10, "threads": 8, "seconds": [8.31, 1.62],
     "speedup": 5.1296296296296, "params": {"z": "last", "a": "first\tline"}},
    {"task": "noisy-grad", "n": 15, "depth": 6, "threads": 1, "seconds": [], "params": {"p": "0.001"}},
    {"task": "single-gate", "n": 33, "depth": 0, "threads": 1, "seconds": [1e16, 3e-300, 0.1, 1 / 3],
     "params": {"gate": "H"}},
]


@pytest.mark.parametrize("fmt", ["json", "csv"])
def test_bench_report_matches_reference_harness(fmt):
    import paper_2406_19212_b200 as vqb
    if not os.path.exists(oracle.REFBENCH_CLI):
        pytest.skip("reference harness not built")
    mine = vqb.device().bench_report(BENCH_RECORDS, fmt)
    theirs = oracle.reference_bench_report(BENCH_RECORDS, fmt)
    assert mine == theirs


def test_bench_report_rejects_empty():
    import paper_2406_19212_b200 as vqb
    from paper_2406_19212_b200.abi import UsageError
    with pytest.raises(UsageError):
        vqb.device().bench_report([], "json")
