"""1- and 2-byte words (uint8 / fp16-bf16) against a same-size copy_:
flushed means of 30 launches, the planner's kernel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_03686_b200 as vp  # noqa: E402
from paper_2506_03686_b200.api import execute_device  # noqa: E402

CASES = [((8192, 8192), (1, 0), 1), ((4096, 4096), (1, 0), 2), ((32, 64, 56, 56), (0, 2, 3, 1), 2),
         ((64, 128, 112, 112), (0, 2, 3, 1), 1), ((17, 9, 13, 15, 11, 27), (5, 2, 0, 4, 1, 3), 2),
         ((4099, 4097), (1, 0), 2), ((2,) * 26, tuple(range(25, -1, -1)), 2), ((128, 64, 32, 512), (2, 0, 1, 3), 2),
         ((8191, 8191), (1, 0), 1), ((512, 512, 27, 9), (1, 0, 2, 3), 1),
         ((64, 512, 7, 7), (0, 2, 3, 1), 2), ((64, 256, 14, 14), (0, 2, 3, 1), 2), ((64, 7, 7, 512), (0, 3, 1, 2), 2),
         ((16, 1024, 12, 64), (0, 2, 1, 3), 2), ((8, 2048, 32, 128), (0, 2, 1, 3), 2), ((3, 1080, 1920), (1, 2, 0), 1),
         ((1024, 1024), (1, 0), 1), ((2048, 1024), (1, 0), 1), ((1000, 1000), (1, 0), 2), ((5000, 3000), (1, 0), 2)]
dev = torch.device("cuda", 0)
fl = bench.Flusher(torch, dev)
st = torch.cuda.current_stream()
for shape, axes, E in CASES:
    n = int(np.prod(shape)) * E
    x = torch.randint(0, 255, (n,), dtype=torch.uint8, device=dev)
    y = torch.empty_like(x)
    p = vp.build_program(vp.TensorLayout.from_shape(shape, E), vp.from_numpy_convention(axes))
    t = np.mean(bench.time_device(torch, lambda: execute_device(p, x, out=y), 30, 3, fl, st)) * 1e3
    dt = {1: torch.uint8, 2: torch.int16}[E]
    xv = x.view(dt).view(shape)
    ok = torch.equal(y.view(dt), xv.permute(axes).reshape(-1)) if len(shape) <= 25 else None
    tc = np.mean(bench.time_device(torch, lambda: y.copy_(x), 30, 3, fl, st)) * 1e3
    vec = [ln for ln in p.text.splitlines() if ln.startswith("vector") or ln.startswith("rows:")][:1]
    print(f"{shape} {axes} E={E} {n / 2**20:6.1f} MiB {p.kernel:5s} {t:8.2f} us  copy_ {tc:7.2f} us  "
          f"{tc / t:.3f} of copy_  parity {ok}  {vec}", flush=True)
