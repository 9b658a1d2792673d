"""B200-native (sm_100a) data-parallel core of the JuliVQC-style simulator.

The native library ``lib/libvqcs_b200.so`` (CUDA kernels + the C-ABI of
include/vqcs_b200.h) is the product; this package is its Python binding.
`device()` fails loudly when the library is missing: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as _ct
import os as _os

from .abi import (ChannelKind, ChannelOp, Circuit, GateKind, GateOp, PauliOperator,  # noqa: F401
                  PauliTerm, heisenberg_1d, make_channel, make_gate, parametric_gate,
                  standard_channel, standard_gate, sum_z)
from .engine import Engine, State  # noqa: F401

HERE = _os.path.dirname(_os.path.abspath(__file__))
LIB_PATH = _os.path.join(HERE, "lib", "libvqcs_b200.so")

_device = None


def library_path() -> str:
    return LIB_PATH


def load_library() -> _ct.CDLL:
    if not _os.path.exists(LIB_PATH):
        raise RuntimeError(f"native library missing: {LIB_PATH} (run __graft_entry__.build())")
    return _ct.CDLL(LIB_PATH)


def device() -> Engine:
    """The CUDA engine (libvqcs_b200.so). Raises if the library is absent."""
    global _device
    if _device is None:
        _device = Engine(load_library(), "vqb_", "b200")
    return _device
