"""One config's hot call, repeated (for ncu: warm the specialised kernels
first, then profile a chosen launch). usage: profile_grad.py <config> [reps]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_19212_b200 as vqb
from paper_2406_19212_b200 import circuits
name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dev = vqb.device()
if name == "noisy15":
    w = circuits.config3()
    s = dev.mixed_state(w.num_qubits)
    run = lambda: dev.gradient_mixed(w.observable, w.circuit, s)
elif name == "qaoa30":
    w = circuits.config2()
    s = dev.pure_state(w.num_qubits)
    run = lambda: dev.gradient_pure(w.observable, w.circuit, s)
elif name == "hea20":
    w = circuits.config0()
    s = dev.pure_state(w.num_qubits)
    run = lambda: dev.gradient_pure(w.observable, w.circuit, s)
else:
    w = circuits.config1()
    s = dev.pure_state(w.num_qubits)
    run = lambda: dev.apply_circuit(w.circuit, s)
for _ in range(reps):
    run()
print("done", name)
