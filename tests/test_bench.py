"""CPU: bench.py's host-side logic (no GPU): workload definitions, the
touched-amplitude byte rule, the bounded reference samples
and their scaling, the clock sampler's fallback."""
import argparse
import math
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def wl(name, world=1):
    return bench.Workload(name, argparse.Namespace(unfused=False), world)


def test_workloads_match_baseline_configs():
    assert (wl("rqc28").n, wl("rqc28").gates, wl("rqc28").kind) == (28, 785, "apply")
    assert (wl("hea20").n, wl("hea20").kind) == (20, "grad_pure")
    assert (wl("qaoa30").n, wl("qaoa30").kind) == (30, "grad_pure")
    assert (wl("noisy15").n, wl("noisy15").mixed, wl("noisy15").kind) == (15, True, "grad_mixed")
    # config 4: 33 + log2(N) qubits, 128 GiB per GPU; sharded only at N > 1
    for world, n in [(1, 33), (2, 34), (4, 35), (8, 36)]:
        w = wl("rqc33", world)
        assert w.n == n and w.sharded == (world > 1)
    assert wl("qaoa30", 2).sharded and not wl("hea20", 2).sharded


def test_touched_amplitude_bytes():
    # every config-1 element is a dense 1- or 2-qubit gate: one full pass each
    w = wl("rqc28")
    assert w.algorithmic_bytes() == pytest.approx(785 * 32.0 * 2 ** 28)
    # per GPU of a sharded run: 2^(n - log2 N) amplitudes
    assert wl("rqc33", 8).algorithmic_bytes(8) == pytest.approx(wl("rqc33", 8).algorithmic_bytes(1) / 8)
    # adjoint: forward + H|psi> + reverse on two states
    g = wl("hea20")
    fwd = g.algorithmic_bytes() / (32.0 * 2 ** 20)
    assert fwd > 3 * 600  # 600 dense rotations forward, twice that reversed


@pytest.mark.parametrize("name,scale", [("rqc28", 1.0), ("hea20", 1.0), ("qaoa30", 2.0 ** -8),
                                        ("noisy15", 4.0 ** -4), ("rqc33", 2.0 ** -5)])
def test_reference_samples_are_bounded_and_scaled(name, scale):
    run, units, sample = bench.reference_sample(wl(name), full=True)
    assert callable(run) and sample
    if name == "rqc28":
        assert units == 160 and "first 160" in sample
    elif name == "rqc33":
        assert units == pytest.approx(160 * scale) and "extrapolated" in sample
    else:
        assert units == pytest.approx(scale)
        if scale != 1.0:
            assert "extrapolated" in sample


def test_clock_sampler_summary_without_samples():
    c = bench.ClockSampler(0)
    assert c.summary()["reasons"] == ["unsampled"]
    c.samples = [(1800.0, 1965.0, {"sw_power_cap"}), (1900.0, 1965.0, set())]
    s = c.summary()
    assert s["sm_mhz"] == pytest.approx(1850.0) and s["sm_max_mhz"] == 1965.0
    assert s["reasons"] == ["sw_power_cap"]


def test_hbm_peak_reads_measured_file():
    peak, kind = bench.hbm_peak()
    assert peak > 1000 and kind in ("measured", "fallback")


def test_sharded_value_counts_one_circuit_per_step():
    """A sharded run processes ONE circuit per step across all ranks (no
    factor N); replicas each process their own."""
    for world in (2, 4, 8):
        w = wl("rqc33", world)
        assert w.sharded and w.job_units(5) == 5 * w.gates
        q = wl("qaoa30", world)
        assert q.sharded and q.job_units(5) == 5
        r = wl("rqc28", world)
        assert not r.sharded and r.job_units(5) == 5 * r.gates * world
    assert wl("rqc28").job_units(3) == 3 * 785


def test_reference_sample_uses_harness_protocol():
    """Allocated once, std::fill reset per run (src/bench.cpp:128-151)."""
    import oracle
    w = bench.Workload("rqc28", argparse.Namespace(unfused=False), 1)
    smp = bench.ReferenceSample(w)
    smp.n = 8  # shrink for the CPU test; the protocol is what is checked
    smp.circ = bench.Circuit(circ_small())
    eng = oracle.restatement()
    smp.prepare(eng)
    h = smp.state.handle
    smp.run(eng)
    a = eng.download(smp.state)
    smp.run(eng)
    assert smp.state.handle == h  # same allocation
    assert (eng.download(smp.state) == a).all()  # reset to |0...0> before each run
    smp.free()


def circ_small():
    from paper_2406_19212_b200 import circuits
    return circuits.config1(rows=2, cols=4, cycles=3).circuit.elements
