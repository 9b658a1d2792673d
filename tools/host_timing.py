import time, os
import paper_2406_19212_b200 as vqb
from paper_2406_19212_b200 import circuits
dev = vqb.device()
w = circuits.config1()
s = dev.create(28)
for i in range(3):
    dev.apply_circuit(w.circuit, s)
import torch
for i in range(3):
    t0 = time.perf_counter(); dev.apply_circuit(w.circuit, s); t1 = time.perf_counter()
    print("wall ms", round((t1-t0)*1e3, 2))
# host-only cost: pack + planning via plan_blocks
t0 = time.perf_counter(); dev.plan_blocks(w.circuit, 28); t1 = time.perf_counter()
print("plan_blocks ms", round((t1-t0)*1e3,2))
t0 = time.perf_counter(); p = w.circuit.pack(); t1 = time.perf_counter()
print("pack ms", round((t1-t0)*1e3,2))
