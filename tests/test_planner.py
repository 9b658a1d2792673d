"""CPU: the fused executor's host logic (stage packing + block fusion,
csrc/plan.cpp) is exported by vqb_plan_blocks without device work. Applying
the exported blocks in order with numpy must reproduce the reference's
apply_circuit (circuit.hpp:110-129) — reordering only commuting operations
and multiplying blocks exactly."""
import numpy as np
import pytest

import paper_2406_19212_b200 as vqb
from paper_2406_19212_b200 import circuits
from paper_2406_19212_b200.abi import Circuit

from helpers import random_channel, random_density, random_gate, random_state


def apply_block(state, n, positions, mat):
    m = len(positions)
    d = 1 << m
    M = mat.reshape(d, d, order="F")
    psi = state.reshape([2] * n, order="F")  # axis j <-> qubit j+1
    axes = [p - 1 for p in positions]
    # local index bit k <-> positions[k]; tensor axes in order (k = m-1 .. 0) for C-order reshape
    t = np.moveaxis(psi, axes[::-1], list(range(m)))
    shp = t.shape
    t = (M @ t.reshape(d, -1)).reshape(shp)
    t = np.moveaxis(t, list(range(m)), axes[::-1])
    return t.reshape(-1, order="F")


def run_blocks(amps, n, blocks):
    s = amps.copy()
    for pos, mat in blocks:
        s = apply_block(s, n, pos, mat)
    return s


@pytest.fixture(scope="module")
def host():
    return vqb.device()  # host-only entry points; no CUDA call is made


@pytest.mark.parametrize("tile_bits,fuse", [(7, 2), (8, 1), (9, 2), (12, 2), (8, 0)])
def test_plan_reproduces_reference(host, orc, tile_bits, fuse):
    rng = np.random.default_rng(tile_bits * 3 + fuse)
    n = 11
    c = Circuit([random_gate(n, rng) for _ in range(250)])
    blocks, stages = host.plan_blocks(c, n, tile_bits=tile_bits, max_support=fuse)
    assert stages >= 1
    if fuse:
        assert len(blocks) < len(c)  # fusion merged something
    amps = random_state(n, rng)
    got = run_blocks(amps, n, blocks)
    r = orc.from_amplitudes(amps)
    orc.apply_circuit(c, r)
    assert np.max(np.abs(got - orc.download(r))) <= 1e-12


def test_plan_density_matrix_program(host, orc):
    rng = np.random.default_rng(3)
    n = 4
    elems = []
    for _ in range(30):
        elems.append(random_channel(n, rng) if rng.integers(2) else random_gate(n, rng, max_targets=2))
    elems.append(circuits.make_channel([2, 3], circuits.depolarizing2_kraus(0.2)))
    c = Circuit(elems)
    blocks, _ = host.plan_blocks(c, n, mixed=True, tile_bits=6, max_support=2)
    rho = random_density(n, rng)
    got = run_blocks(rho, 2 * n, blocks)
    r = orc.from_amplitudes(rho, True)
    orc.apply_circuit(c, r)
    assert np.max(np.abs(got - orc.download(r))) <= 1e-12


def test_rqc28_stage_count(host):
    """Config 1: 785 gates pack into few HBM passes with 12-bit tiles."""
    w = circuits.config1()
    blocks, stages = host.plan_blocks(w.circuit, 28, tile_bits=12, max_support=2)
    assert stages <= 40
    assert len(blocks) < 785 * 0.6


def test_qaoa_cost_layer_fuses_to_diagonals(host):
    """CNOT Rz CNOT (exp(-i g Z_i Z_j)) multiplies to a diagonal block."""
    w = circuits.config2(n=12, p=1)
    blocks, _ = host.plan_blocks(w.circuit, 12, tile_bits=12, max_support=2)
    diag = 0
    for pos, mat in blocks:
        d = 1 << len(pos)
        M = mat.reshape(d, d, order="F")
        if len(pos) == 2 and np.allclose(M, np.diag(np.diag(M))):
            diag += 1
    assert diag >= len(w.extra["edges"]) // 2
