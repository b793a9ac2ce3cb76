"""PCIe duplex steady state: K back-to-back 2 GiB steps, chunked copies on
1 or 2 streams per direction (what the host pipeline can reach)."""
import time

import torch

n = 2 << 30
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = [torch.empty(n, dtype=torch.uint8).pin_memory() for _ in range(2)]
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")


def run(chunks, nstreams, K=6):
    hs = [torch.cuda.Stream() for _ in range(nstreams)]
    ds = [torch.cuda.Stream() for _ in range(nstreams)]
    c = n // chunks

    def step(k):
        for j in range(chunks):
            with torch.cuda.stream(hs[j % nstreams]):
                d_a[j * c:(j + 1) * c].copy_(h_in[j * c:(j + 1) * c], non_blocking=True)
            with torch.cuda.stream(ds[j % nstreams]):
                h_out[k % 2][j * c:(j + 1) * c].copy_(d_b[j * c:(j + 1) * c], non_blocking=True)
    step(0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(K):
        step(k)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / K
    print(f"chunks {chunks:3d} streams/dir {nstreams}: {2 * n / dt / 1e9:.1f} GB/s duplex", flush=True)


for chunks in (1, 8, 32):
    for ns in (1, 2, 4):
        if ns <= chunks:
            run(chunks, ns)
