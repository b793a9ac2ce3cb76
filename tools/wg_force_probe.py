"""Gather W blocks forced (VPG_WG=2) vs the cost model's choice on shapes
where they apply but the model keeps scalar stores; flushed means of 20,
plans rebuilt in-process (the knob is read at plan creation)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_03686_b200 as vp  # noqa: E402
from paper_2506_03686_b200.api import execute_device  # noqa: E402

CASES = [((64, 2048, 7, 7), (0, 2, 3, 1), E) for E in (1, 2, 4, 8)] + [
    ((64, 512, 14, 14), (0, 2, 3, 1), 2), ((32, 1024, 9, 9), (0, 2, 3, 1), 2), ((8, 32, 2048, 128), (0, 1, 3, 2), 1),
    ((64, 1024, 1000), (0, 2, 1), 2), ((64, 1024, 1000), (0, 2, 1), 4), ((16, 18, 38, 64), (2, 1, 0, 3), 2),
    ((17, 9, 13, 15, 11, 32), (5, 2, 0, 4, 1, 3), 2)]
dev = torch.device("cuda", 0)
fl = bench.Flusher(torch, dev)
st = torch.cuda.current_stream()
for shape, axes, E in CASES:
    n = int(np.prod(shape)) * E
    x = torch.randint(0, 255, (n,), dtype=torch.uint8, device=dev)
    y = torch.empty_like(x)
    res = []
    for wg in ("1", "2"):
        os.environ["VPG_WG"] = wg
        vp.program_cache_clear()
        p = vp.build_program(vp.TensorLayout.from_shape(shape, E), vp.from_numpy_convention(axes))
        t = np.mean(bench.time_device(torch, lambda: execute_device(p, x, out=y), 20, 3, fl, st)) * 1e3
        res.append((t, "gather" in p.text))
    tc = np.mean(bench.time_device(torch, lambda: y.copy_(x), 20, 3, fl, st)) * 1e3
    print(f"{shape} {axes} E={E}: model {res[0][0]:7.2f} us (gather {res[0][1]}, {tc / res[0][0]:.3f}) | "
          f"forced {res[1][0]:7.2f} us (gather {res[1][1]}, {tc / res[1][0]:.3f})", flush=True)
