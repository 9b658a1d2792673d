"""Small invocations of every kernel family for compute-sanitizer (memcheck,
racecheck, synccheck): the interpreter and the specialised (NVRTC) stage
kernels forward and adjoint, pure and density-matrix, reductions, measurement.
Run by tools/sanitize.sh on the GPU box; sizes are small so the instrumented
run finishes in minutes."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2406_19212_b200 as vqb  # noqa: E402
from paper_2406_19212_b200 import circuits  # noqa: E402
from paper_2406_19212_b200.abi import sum_z  # noqa: E402

dev = vqb.device()
for jit in ("0", "1"):
    os.environ["VQB_JIT"] = jit
    w = circuits.config1(rows=3, cols=4, cycles=6)
    s = dev.pure_state(12)
    dev.apply_circuit(w.circuit, s)
    print("rqc12", jit, dev.norm(s), dev.expectation(sum_z(12), s))
    dev.measure(s, 3, 0.4)
    g = circuits.config0(n=12, layers=2)
    print("hea12", jit, dev.gradient_pure(g.observable, g.circuit, dev.pure_state(12))[0])
    q = circuits.config2(n=12, p=2)
    print("qaoa12", jit, dev.gradient_pure(q.observable, q.circuit, dev.pure_state(12))[0])
    d = circuits.config3(n=6, layers=2)
    print("noisy6", jit, dev.gradient_mixed(d.observable, d.circuit, dev.mixed_state(6))[0])
os.environ["VQB_JIT"] = "1"
os.environ["VQB_REV_REGS"] = "16"
q = circuits.config2(n=12, p=2)
print("qaoa12 r16", dev.gradient_pure(q.observable, q.circuit, dev.pure_state(12))[0])
print("sanitize probe done")
