"""PCIe ceiling on this box: pinned H2D, D2H, and both concurrently (2 GiB)."""
import time

import torch

n = 2 << 30
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(f, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


h2d = t(lambda: d_a.copy_(h_in, non_blocking=True))
d2h = t(lambda: h_out.copy_(d_b, non_blocking=True))


def both():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)


bb = t(both)
print(f"H2D {n/h2d/1e9:.1f} GB/s  D2H {n/d2h/1e9:.1f} GB/s  concurrent {2*n/bb/1e9:.1f} GB/s total "
      f"({bb*1e3:.1f} ms for 2x2 GiB)")
# chunked 2-D pattern like the cfg5 pipeline: 128 KiB rows
rows = 16384
w = 128 << 10
t2 = t(lambda: torch.cuda.cudart().cudaMemcpy2DAsync if False else d_a[: rows * w].copy_(h_in[: rows * w], non_blocking=True))
print(f"H2D 2 GiB as one copy again {rows*w/t2/1e9:.1f} GB/s")
