"""Time a fixed list of shapes with the library VPG_LIB_PATH names (same-box
A/B of library builds: run once per build, join the lines by shape).
    python tools/lib_ab.py shapes.txt      # lines: SHAPE | AXES | E
"""
import ast
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_03686_b200 as vp  # noqa: E402
from paper_2506_03686_b200.api import execute_device  # noqa: E402

dev = torch.device("cuda", 0)
fl = bench.Flusher(torch, dev)
st = torch.cuda.current_stream()
for line in open(sys.argv[1]):
    if not line.strip() or line.startswith("#"):
        continue
    sh, ax, e = line.split("|")
    shape, axes, E = ast.literal_eval(sh.strip()), ast.literal_eval(ax.strip()), int(e)
    nbytes = int(np.prod(shape)) * E
    x = torch.randint(0, 255, (nbytes,), dtype=torch.uint8, device=dev)
    y = torch.empty_like(x)
    p = vp.build_program(vp.TensorLayout.from_shape(shape, E), vp.from_numpy_convention(axes))
    ts = []
    for rep in range(3):
        t = bench.time_device(torch, lambda: execute_device(p, x, out=y), 9, 3, fl, st)
        ts.append(sorted(t)[4] * 1e3)
    tc = sorted(bench.time_device(torch, lambda: y.copy_(x), 9, 3, fl, st))[4] * 1e3
    print(f"{shape}|{axes}|{E}|{np.mean(ts):.1f}|{tc / np.mean(ts):.3f}", flush=True)
    del x, y
