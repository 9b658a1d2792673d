"""GPU: the reference-side C++ binding (include/vqcs_b200.hpp) used from a
program written against the reference's own API (tests/cpp/facade_demo.cpp):
vqcs:: (CPU reference) and vqb:: (B200) agree, and library errors surface as
the reference's exception classes."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
EXE = os.path.join(os.path.dirname(__file__), "cpp", "_build", "facade_demo")


@pytest.mark.skipif(not os.path.exists(EXE), reason="facade demo not built (needs /root/reference)")
def test_cpp_facade_drop_in():
    out = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    print(out.stdout, out.stderr)
    assert out.returncode == 0, out.stdout + out.stderr
