"""A/B planner env settings on one shape: python tools/shape_ab.py 'SHAPE' 'AXES' E 'ENV=a|ENV=b'"""
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
variants = sys.argv[4].split("|")
dev = torch.device("cuda", 0)
fl = bench.Flusher(torch, dev)
st = torch.cuda.current_stream()
nbytes = int(np.prod(shape)) * E
x = torch.randint(0, 255, (nbytes,), dtype=torch.uint8, device=dev)
y = torch.empty_like(x)
progs = {}
for v in variants:
    k, val = v.split("=")
    os.environ[k] = val
    vp.program_cache_clear()
    progs[v] = vp.build_program(vp.TensorLayout.from_shape(shape, E), vp.from_numpy_convention(axes))
    del os.environ[k]
res = {v: [] for v in variants}
for rep in range(5):
    for v in variants:
        t = bench.time_device(torch, lambda: execute_device(progs[v], x, out=y), 11, 3, fl, st)
        res[v].append(sorted(t)[5] * 1e3)
tc = bench.time_device(torch, lambda: y.copy_(x), 11, 3, fl, st)
c = sorted(tc)[5] * 1e3
for v in variants:
    m = progs[v].metadata
    print(f"{v:24s} runs {m['src_run']}x{m['dst_run']} T={m['tile_elems']}: mean {np.mean(res[v]):7.1f} us "
          f"({c / np.mean(res[v]):.3f} of copy_ {c:.1f} us)")
