"""Planning-only run on a host without a GPU (VQB_DRYRUN=1): lowers one
gradient / circuit of a BASELINE config and dumps every generated kernel and
its lowered program (VQB_JIT_DUMP) for tools/jit_inspect.py.
usage: dryrun_dump.py <hea20|qaoa30|noisy15|rqc28|rqc33> <out dir>"""
import os
import sys

os.environ["VQB_DRYRUN"] = "1"
os.environ["VQB_JIT_DUMP"] = sys.argv[2]
os.environ.setdefault("VQB_PARALLEL_ADJOINT", "0")
os.makedirs(sys.argv[2], exist_ok=True)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_19212_b200 as vqb  # noqa: E402
from paper_2406_19212_b200 import circuits  # noqa: E402

name = sys.argv[1]
w = {"hea20": circuits.config0, "qaoa30": circuits.config2, "noisy15": circuits.config3,
     "rqc28": circuits.config1, "rqc33": lambda: circuits.config4(1)}[name]()
dev = vqb.device()
s0 = dev.create(w.num_qubits, w.mixed)
if name.startswith("rqc"):
    dev.apply_circuit(w.circuit, s0)
else:
    (dev.gradient_mixed if w.mixed else dev.gradient_pure)(w.observable, w.circuit, s0)
print(len(os.listdir(sys.argv[2])), "files")
