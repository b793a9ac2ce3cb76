"""Time the first K tile candidates of one shape (flushed launches)."""
import ast
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_03686_b200 as vp  # noqa: E402
from paper_2506_03686_b200.api import execute_device  # noqa: E402

shape, axes, E = ast.literal_eval(sys.argv[1]), ast.literal_eval(sys.argv[2]), int(sys.argv[3])
K = int(sys.argv[4]) if len(sys.argv) > 4 else 10
dev = torch.device("cuda", 0)
fl = bench.Flusher(torch, dev)
st = torch.cuda.current_stream()
nbytes = int(np.prod(shape)) * E
x = torch.randint(0, 255, (nbytes,), dtype=torch.uint8, device=dev)
y = torch.empty_like(x)
lay, pm = vp.TensorLayout.from_shape(shape, E), vp.from_numpy_convention(axes)
tc = bench.time_device(torch, lambda: y.copy_(x), 11, 3, fl, st)
c = sorted(tc)[5] * 1e3
for k in range(K):
    try:
        p = vp.build_program(lay, pm, candidate=k)
    except vp.LayoutError:
        break
    t = bench.time_device(torch, lambda: execute_device(p, x, out=y), 11, 3, fl, st)
    us = sorted(t)[5] * 1e3
    m = p.metadata
    vec = [ln for ln in p.text.splitlines() if ln.startswith("vector")][0]
    print(f"cand {k}: {m['src_run']}x{m['dst_run']} T={m['tile_elems']} pitch {m['smem_pitch']} {vec} "
          f"-> {us:6.1f} us ({c / us:.3f} of copy_)", flush=True)
