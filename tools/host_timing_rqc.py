"""Host-side phase timing of config-1 apply_circuit (VQB_HOST_TIMING=1)."""
import time
import paper_2406_19212_b200 as vqb
from paper_2406_19212_b200 import circuits
dev = vqb.device()
w = circuits.config1()
s = dev.pure_state(28)
for i in range(4):
    t0 = time.perf_counter()
    dev.apply_circuit(w.circuit, s)
    print("call", i, "%.3f ms" % (1e3 * (time.perf_counter() - t0)), flush=True)
# same call under per-kernel event timing
dev.profile_begin()
t0 = time.perf_counter()
dev.apply_circuit(w.circuit, s)
t1 = time.perf_counter()
prof = dev.profile_end()
print("profiled call wall %.3f ms, kernel sum %.3f ms" % (1e3 * (t1 - t0), sum(v[1] for v in prof.values())), prof)
