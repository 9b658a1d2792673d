import sys, time, ctypes as ct
sys.path.insert(0, '/root/repo')
import torch
import paper_2406_19212_b200 as vqb
from paper_2406_19212_b200 import circuits
from paper_2406_19212_b200.abi import c128_p
eng = vqb.device()
w = circuits.config0()
st = eng.create(20, False)
h = torch.zeros(2 << 20, dtype=torch.float64, pin_memory=True); h[0] = 1
pin = ct.cast(ct.c_void_p(h.data_ptr()), c128_p)
up = eng._fn("state_upload")
for _ in range(5): eng.gradient_pure(w.observable, w.circuit, st)
def t(f, n=50):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(n): f()
    return (time.perf_counter() - t0) / n * 1e3
print("grad only %.3f ms" % t(lambda: eng.gradient_pure(w.observable, w.circuit, st)))
print("upload only %.3f ms" % t(lambda: eng.check(up(st.handle, pin, ct.c_uint64(1 << 20)))))
print("upload+grad %.3f ms" % t(lambda: (eng.check(up(st.handle, pin, ct.c_uint64(1 << 20))), eng.gradient_pure(w.observable, w.circuit, st))))
print("set_zero+grad %.3f ms" % t(lambda: (eng.check(eng._fn("state_set_zero")(st.handle)), eng.gradient_pure(w.observable, w.circuit, st))))
