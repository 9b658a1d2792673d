"""Host-side phase timing of one config-0 gradient (VQB_HOST_TIMING=1)."""
import time
import paper_2406_19212_b200 as vqb
from paper_2406_19212_b200 import circuits
dev = vqb.device()
w = circuits.config0()
s0 = dev.pure_state(20)
for i in range(4):
    t0 = time.perf_counter()
    dev.gradient_pure(w.observable, w.circuit, s0)
    print("call", i, "%.3f ms" % (1e3 * (time.perf_counter() - t0)), flush=True)
