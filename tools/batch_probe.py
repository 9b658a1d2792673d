"""Slope of vqb_apply_circuit_copy_batch time over the job count (config 1)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2406_19212_b200 as vqb
from paper_2406_19212_b200 import circuits
dev = vqb.device()
w = circuits.config1()
n = 28
h_in = torch.zeros(2 << n, dtype=torch.float64, pin_memory=True); h_in[0] = 1
outs = [torch.empty(2 << n, dtype=torch.float64, pin_memory=True) for _ in range(3)]
mode = sys.argv[1] if len(sys.argv) > 1 else "full"
for jobs in [1, 2, 4, 8, 16]:
    ins = [h_in.data_ptr()] * jobs
    o = [outs[j % 3].data_ptr() for j in range(jobs)]
    dev.apply_circuit_copy_batch(w.circuit, n, ins[:1], o[:1])
    torch.cuda.synchronize()
    t = time.perf_counter()
    dev.apply_circuit_copy_batch(w.circuit, n, ins, o)
    dt = time.perf_counter() - t
    print(f"jobs {jobs:2d}: {dt*1e3:8.1f} ms  {dt*1e3/jobs:6.1f} ms/job", flush=True)
