"""Cold-start cost of the specialised kernels: first call (compile) vs warm."""
import time
import paper_2406_19212_b200 as vqb
from paper_2406_19212_b200 import circuits
dev = vqb.device()
for name, w in (("rqc28", circuits.config1()), ("qaoa30_fwd", circuits.config2())):
    s = dev.create(w.num_qubits)
    for i in range(3):
        t0 = time.perf_counter()
        dev.apply_circuit(w.circuit, s)
        print(name, "call", i, "%.3f s" % (time.perf_counter() - t0), flush=True)
    s.free()
