"""Tiny permutations (1-8 MiB) against a same-size copy_: flushed means of
30 launches, planner default vs VPG_TINY=0 (run twice, once per setting:
the knob is read at plan creation).  `jit` as argv[1]: specialised
(NVRTC) kernel vs the ahead-of-time kernel instead."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_03686_b200 as vp  # noqa: E402
from paper_2506_03686_b200.api import execute_device  # noqa: E402

CASES = [((1024, 1024), (1, 0), 1), ((2048, 1024), (1, 0), 1), ((64, 512, 7, 7), (0, 2, 3, 1), 2),
         ((64, 7, 7, 512), (0, 3, 1, 2), 2), ((1000, 1000), (1, 0), 2), ((512, 512), (1, 0), 4),
         ((1024, 1024), (1, 0), 4), ((32, 256, 14, 14), (0, 2, 3, 1), 4), ((17, 9, 13, 15, 11), (4, 2, 0, 3, 1), 4),
         ((256, 1024), (1, 0), 8), ((2,) * 20, tuple(range(19, -1, -1)), 4)]
dev = torch.device("cuda", 0)
fl = bench.Flusher(torch, dev)
st = torch.cuda.current_stream()
for shape, axes, E in CASES:
    n = int(np.prod(shape)) * E
    x = torch.randint(0, 255, (n,), dtype=torch.uint8, device=dev)
    y = torch.empty_like(x)
    res = []
    knob = "VPG_JIT" if len(sys.argv) > 1 and sys.argv[1] == "jit" else "VPG_TINY"
    for tiny in ("1", "0"):
        os.environ[knob] = tiny
        vp.program_cache_clear()
        p = vp.build_program(vp.TensorLayout.from_shape(shape, E), vp.from_numpy_convention(axes))
        t = np.mean(bench.time_device(torch, lambda: execute_device(p, x, out=y), 30, 3, fl, st)) * 1e3
        res.append((t, p.metadata.get("tile_elems"), p.kernel))
    tc = np.mean(bench.time_device(torch, lambda: y.copy_(x), 30, 3, fl, st)) * 1e3
    print(f"{shape} {axes} E={E} {n / 2**20:5.1f} MiB copy_ {tc:6.2f} us | {knob}=1 {res[0][0]:6.2f} us "
          f"(T={res[0][1]}, {tc / res[0][0]:.3f}) | {knob}=0 {res[1][0]:6.2f} us (T={res[1][1]}, {tc / res[1][0]:.3f})",
          flush=True)
