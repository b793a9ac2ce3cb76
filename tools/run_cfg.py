"""Run one BASELINE config's permutation a few times (for ncu / sanitizers)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2506_03686_b200 import TensorLayout, build_program, from_numpy_convention  # noqa: E402
from paper_2506_03686_b200.api import execute_device  # noqa: E402
from paper_2506_03686_b200.workloads import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="cfg5")
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--force", default=None)
a = ap.parse_args()
for cfg in a.cfg.split(","):
    wl = CONFIGS[cfg]
    prog = build_program(TensorLayout.from_shape(wl.shape, wl.elem_bytes), from_numpy_convention(wl.axes),
                         force=a.force)
    print(cfg, prog.text, flush=True)
    n = wl.numel * wl.elem_bytes
    x = torch.randint(0, 255, (n,), dtype=torch.uint8, device="cuda")
    y = torch.empty_like(x)
    for _ in range(a.iters):
        execute_device(prog, x, out=y)
    torch.cuda.synchronize()
print("done")
