"""Flushed single-launch timing: specialised (JIT) vs ahead-of-time kernel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2506_03686_b200 import TensorLayout, build_program, from_numpy_convention  # noqa: E402
from paper_2506_03686_b200.api import execute_device  # noqa: E402
from paper_2506_03686_b200.workloads import CONFIGS  # noqa: E402

dev = torch.device("cuda", 0)
fl = bench.Flusher(torch, dev)
st = torch.cuda.current_stream()
for k in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["cfg1", "cfg2", "cfg3", "cfg5"]):
    wl = CONFIGS[k]
    n = wl.numel * wl.elem_bytes
    x = torch.randint(0, 255, (n,), dtype=torch.uint8, device=dev)
    y = torch.empty_like(x)
    res = {}
    for rep in range(3):
        for jit in (False, True):
            prog = build_program(TensorLayout.from_shape(wl.shape, wl.elem_bytes), from_numpy_convention(wl.axes),
                                 jit=jit)
            t = bench.time_device(torch, lambda: execute_device(prog, x, out=y), 20, 3, fl, st)
            res.setdefault(jit, []).append(sorted(t)[10] * 1e3)
    print(k, {("jit" if j else "aot"): [round(v, 1) for v in vs] for j, vs in res.items()}, flush=True)
