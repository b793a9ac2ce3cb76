"""Stride-1-preserving permutations with odd row lengths: the rows kernel
(word-width vectors) against the tile kernel (forced), flushed means of 30
launches, same-size copy_ beside them."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_03686_b200 as vp  # noqa: E402
from paper_2506_03686_b200.api import execute_device  # noqa: E402

CASES = [((36, 1060, 439), (1, 0, 2), 8), ((20, 150, 4099), (1, 0, 2), 8), ((40, 300, 1023), (1, 0, 2), 4),
         ((256, 384, 129), (1, 0, 2), 4), ((300, 200, 257), (1, 0, 2), 8), ((64, 70, 2049), (1, 0, 2), 8),
         ((3, 5, 7, 11, 13, 17, 19), (1, 0, 3, 2, 4, 5, 6), 8), ((100, 100, 1001), (1, 0, 2), 4)]
if len(sys.argv) > 1 and sys.argv[1] == "sweep":
    # 8-byte words, row lengths not a multiple of 16 bytes, two outer layouts
    CASES = []
    for L in (65, 129, 257, 439, 1001, 2049, 4099, 8193, 16385):
        per = (96 << 20) // (8 * L)
        a = int(max(2, round((per / 3) ** 0.5)))
        b = max(2, per // a)
        CASES.append(((a, b, L), (1, 0, 2), 8))
        c = max(2, int(round(per ** (1 / 3))))
        CASES.append(((c, max(2, per // (c * c)), c, L), (2, 0, 1, 3), 8))
if len(sys.argv) > 1 and sys.argv[1] == "sweep16":
    # rows that ARE a multiple of 16 bytes (rows kernel / TMA bulk rows today)
    CASES = []
    for E in (4, 8):
        for rb in (512, 1024, 2048, 4096, 16384):
            L = rb // E
            per = (96 << 20) // (E * L)
            a = int(max(2, round((per / 3) ** 0.5)))
            CASES.append(((a, max(2, per // a), L), (1, 0, 2), E))
            c = max(2, int(round(per ** (1 / 3))))
            CASES.append(((c, max(2, per // (c * c)), c, L), (2, 0, 1, 3), E))
dev = torch.device("cuda", 0)
fl = bench.Flusher(torch, dev)
st = torch.cuda.current_stream()
for shape, axes, E in CASES:
    n = int(np.prod(shape)) * E
    x = torch.randint(0, 255, (n,), dtype=torch.uint8, device=dev)
    y = torch.empty_like(x)
    res = {}
    for force in (None, "tile"):
        p = vp.build_program(vp.TensorLayout.from_shape(shape, E), vp.from_numpy_convention(axes), force=force)
        t = np.mean(bench.time_device(torch, lambda: execute_device(p, x, out=y), 30, 3, fl, st)) * 1e3
        tdt = {4: torch.int32, 8: torch.int64}[E]
        ok = bench.sample_parity(torch, x.view(tdt), y.view(tdt), shape, axes, nsamp=1 << 16)
        res[force or "planner"] = (p.kernel, t, ok)
    tc = np.mean(bench.time_device(torch, lambda: y.copy_(x), 30, 3, fl, st)) * 1e3
    print(f"{shape} {axes} E={E} {n / 2**20:6.1f} MiB copy_ {tc:7.2f} us | "
          + " | ".join(f"{k}: {v[0]} {v[1]:7.2f} us ({tc / v[1]:.3f} of copy_, parity {v[2]})" for k, v in res.items()),
          flush=True)
