"""Host-side phase timing of one gradient (VQB_HOST_TIMING=1).
usage: host_timing_grad.py [hea20|qaoa30|noisy15]"""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_19212_b200 as vqb  # noqa: E402
from paper_2406_19212_b200 import circuits  # noqa: E402
name = sys.argv[1] if len(sys.argv) > 1 else "hea20"
dev = vqb.device()
if name == "qaoa30":
    w = circuits.config2()
elif name == "noisy15":
    w = circuits.config3()
else:
    w = circuits.config0()
s0 = dev.create(w.num_qubits, w.mixed)
fn = dev.gradient_mixed if w.mixed else dev.gradient_pure
for i in range(4):
    t0 = time.perf_counter()
    fn(w.observable, w.circuit, s0)
    print("call", i, "%.3f ms" % (1e3 * (time.perf_counter() - t0)), flush=True)
