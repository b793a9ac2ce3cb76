"""Stride-1-preserving permutations (rows kernel, K1) with row lengths that
are not a multiple of 16 bytes, against a same-size copy_ (flushed single
launches, mean of 30) -- how far the per-element-width row walk is from a
16-byte copy.   usage: python tools/rows_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_03686_b200 as vp  # noqa: E402
from paper_2506_03686_b200.api import execute_device  # noqa: E402

CASES = [
    ((64, 32, 1023, 4), (1, 0, 2, 3), 4),
    ((36, 1060, 439), (1, 0, 2), 8),
    ((128, 64, 7, 13, 8), (1, 0, 2, 3, 4), 4),
    ((512, 512, 27, 3), (1, 0, 2, 3), 4),
    ((1000, 300, 9, 5), (1, 0, 2, 3), 8),
    ((17, 9, 13, 15, 11, 27), (2, 0, 1, 4, 3, 5), 4),
    ((256, 384, 129), (1, 0, 2), 4),
    ((4096, 2, 2050), (1, 0, 2), 8),
    ((64, 32, 1024, 4), (1, 0, 2, 3), 4),
    ((40, 300, 1023), (1, 0, 2), 4),
    ((20, 150, 4099), (1, 0, 2), 8),
    ((3000, 50, 77), (1, 0, 2), 4),
]
dev = torch.device("cuda", 0)
fl = bench.Flusher(torch, dev)
st = torch.cuda.current_stream()
for shape, axes, E in CASES:
    n = int(np.prod(shape)) * E
    x = torch.randint(0, 255, (n,), dtype=torch.uint8, device=dev)
    y = torch.empty_like(x)
    p = vp.build_program(vp.TensorLayout.from_shape(shape, E), vp.from_numpy_convention(axes))
    t = np.mean(bench.time_device(torch, lambda: execute_device(p, x, out=y), 30, 3, fl, st)) * 1e3
    tdt = {4: torch.int32, 8: torch.int64}[E]
    ok = bench.sample_parity(torch, x.view(tdt), y.view(tdt), shape, axes, nsamp=1 << 16)
    tc = np.mean(bench.time_device(torch, lambda: y.copy_(x), 30, 3, fl, st)) * 1e3
    rows = [ln for ln in p.text.splitlines() if ln.startswith("rows")][-1:]
    print(f"{shape} {axes} E={E} {p.kernel:5s} {n / 2**20:7.1f} MiB: {t:8.2f} us  copy_ {tc:8.2f} us  "
          f"{tc / t:.3f} of copy_  {2 * n / t / 1e3:6.0f} GB/s  parity {ok}  {rows[:1]}", flush=True)
