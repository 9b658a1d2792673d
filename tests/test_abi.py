"""CPU: the C-ABI boundary — every symbol include/vqcs_b200.h declares is exported
by libvqcs_b200.so (loaded without a GPU; no compute calls), the oracle
libraries implement the same entry points, and the ctypes struct layouts
match the C header."""
import ctypes as ct
import os
import re
import subprocess

import pytest

import oracle
import paper_2406_19212_b200 as vqb
from paper_2406_19212_b200 import abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "vqcs_b200.h")


def declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"VQB_API\s+[\w\s\*]+?\b(vqb_\w+)\s*\(", text)))


def test_header_declares_the_path():
    names = declared()
    for must in ["vqb_apply_gate", "vqb_apply_circuit", "vqb_apply_channel", "vqb_expectation",
                 "vqb_apply_operator", "vqb_reverse_step", "vqb_gradient_pure",
                 "vqb_gradient_mixed", "vqb_bilinear_form", "vqb_state_create", "vqb_plan_blocks"]:
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = vqb.load_library()
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", vqb.library_path()], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r" T (vqb_\w+)", out))
    assert set(declared()) <= exported
    # nothing but the ABI leaks out of the shared object
    assert all(n.startswith("vqb_") for n in exported)


def test_oracles_implement_the_same_entry_points():
    core = [n[len("vqb_"):] for n in declared()
            if n[len("vqb_"):] in set(abi.ABI_FUNCTIONS) - {
                "build_info", "kernel_launch_count", "flop_count", "debug_jit_source", "profile_begin", "profile_end",
                "state_stream",
                "state_wrap", "state_device_ptr", "state_set_zero", "apply_circuit_unfused",
                "apply_circuit_copy_batch", "plan_blocks"}]
    libs = [("vqcsorc_", ct.CDLL(oracle.ORC_SO), set())]
    if oracle.reference_available():
        # the reference draws measurement outcomes from a std::mt19937_64 it is
        # handed, so its shim exposes measure_seeded/uniform_unit instead
        libs.append(("vqcsref_", ct.CDLL(oracle.REF_SO),
                     {"measure", "measure_probability", "collapse"}))
    for prefix, lib, exempt in libs:
        missing = [c for c in core if c not in exempt and not hasattr(lib, prefix + c)]
        assert not missing, (prefix, missing)
    if oracle.reference_available():
        ref = ct.CDLL(oracle.REF_SO)
        assert hasattr(ref, "vqcsref_measure_seeded") and hasattr(ref, "vqcsref_uniform_unit")


def test_struct_layouts_match_header():
    src = r"""
#include <stdio.h>
#include <stddef.h>
#include "vqcs_b200.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu\n", sizeof(vqb_op), offsetof(vqb_op, matrix),
         offsetof(vqb_op, kraus), sizeof(vqb_pauli_term), offsetof(vqb_pauli_term, labels),
         sizeof(vqb_c128));
  return 0;
}
"""
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "l.c")
        open(c, "w").write(src)
        exe = os.path.join(d, "l")
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe], check=True)
        got = list(map(int, subprocess.run([exe], capture_output=True, text=True).stdout.split()))
    want = [ct.sizeof(abi.vqb_op), abi.vqb_op.matrix.offset, abi.vqb_op.kraus.offset,
            ct.sizeof(abi.vqb_pauli_term), abi.vqb_pauli_term.labels.offset, ct.sizeof(abi.c128)]
    assert got == want


def test_status_codes_map_to_reference_exceptions():
    # errors.hpp:23-96 declaration order
    names = ["SizeError", "ShapeError", "ValidityError", "DomainError", "IndexError_",
             "TypeError_", "UnsupportedError", "DegenerateStateError",
             "NonInvertibleChannelError", "IoError", "UsageError"]
    for code, name in enumerate(names, start=1):
        assert abi.STATUS_TO_ERROR[code].__name__ == name


def test_host_gate_algebra_matches_reference(ref):
    """vqb_gate_matrix / derivative / inverse / channel_superop are host-only:
    callable without a GPU, and equal to the reference's gates.hpp."""
    import numpy as np
    from paper_2406_19212_b200.abi import GateKind, parametric_gate, standard_channel, ChannelKind
    dev = vqb.device()
    for g in [parametric_gate(GateKind.Fsim, [1, 2], [0.3, -0.2, 0.1, 0.5, -0.7], [True] * 5),
              parametric_gate(GateKind.CRy, [2, 1], 0.8, True),
              parametric_gate(GateKind.Rz, [3], -1.1, True)]:
        assert np.max(np.abs(dev.gate_matrix(g) - ref.gate_matrix(g))) <= 1e-15
        assert np.max(np.abs(dev.gate_inverse(g) - ref.gate_inverse(g))) <= 1e-15
        for p in range(len(g.params)):
            assert np.max(np.abs(dev.gate_derivative(g, p) - ref.gate_derivative(g, p))) <= 1e-15
    for kind in (ChannelKind.AmplitudeDamping, ChannelKind.PhaseDamping, ChannelKind.Depolarizing):
        ch = standard_channel(kind, 2, 0.37)
        assert np.max(np.abs(dev.channel_superop(ch) - ref.channel_superop(ch))) <= 1e-15
