"""cProfile of one sharded step at world size 1 (config 4 forward) on the GPU."""
import cProfile
import os
import pstats
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2406_19212_b200 as vqb  # noqa: E402
from paper_2406_19212_b200 import circuits  # noqa: E402
from paper_2406_19212_b200.distributed import DeviceEngine, ShardedState  # noqa: E402


class NoDist:
    pass


eng = vqb.device()
w = circuits.config4(num_gpus=1)
st = ShardedState(w.num_qubits, NoDist(), DeviceEngine(eng),
                  torch.zeros(1 << w.num_qubits, dtype=torch.complex128, device="cuda"), 0, 1)
for i in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    st.set_zero()
    st.apply_circuit(w.circuit)
    torch.cuda.synchronize()
    print("step %.1f ms" % ((time.perf_counter() - t) * 1e3), flush=True)
pr = cProfile.Profile()
pr.enable()
st.set_zero()
st.apply_circuit(w.circuit)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(14)
del st
torch.cuda.empty_cache()
s = eng.create(w.num_qubits)
for i in range(2):
    torch.cuda.synchronize()
    t = time.perf_counter()
    eng.check(eng._fn("state_set_zero")(s.handle))
    eng.apply_circuit(w.circuit, s)
    torch.cuda.synchronize()
    print("direct step %.1f ms" % ((time.perf_counter() - t) * 1e3), flush=True)
