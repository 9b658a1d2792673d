"""Host<->device copy rates for the e2e path: 4 GiB pinned H2D, D2H, and both
directions at once on two streams (is the link full duplex here?)."""
import time
import torch
n = 1 << 29  # float64 elements = 4 GiB
h1 = torch.ones(n, dtype=torch.float64, pin_memory=True)
h2 = torch.empty(n, dtype=torch.float64, pin_memory=True)
d1 = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.ones(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
gb = n * 8 / 1e9
for rep in range(2):
    torch.cuda.synchronize(); t = time.perf_counter()
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    torch.cuda.synchronize(); a = time.perf_counter() - t
    t = time.perf_counter()
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize(); b = time.perf_counter() - t
    t = time.perf_counter()
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize(); c = time.perf_counter() - t
    print(f"H2D {gb/a:.1f} GB/s  D2H {gb/b:.1f} GB/s  both {2*gb/c:.1f} GB/s total ({c*1e3:.1f} ms for both)")
