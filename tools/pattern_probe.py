"""Kernel time vs input byte pattern (device-written inputs), cfg5 plan."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_03686_b200 as vp  # noqa: E402
from paper_2506_03686_b200.api import execute_device  # noqa: E402
from paper_2506_03686_b200.workloads import CONFIGS  # noqa: E402

wl = CONFIGS["cfg5"]
dev = torch.device("cuda", 0)
fl = bench.Flusher(torch, dev)
st = torch.cuda.current_stream()
n = wl.numel * wl.elem_bytes
p = vp.build_program(vp.TensorLayout.from_shape(wl.shape, 8), vp.from_numpy_convention(wl.axes))
x = torch.empty(n, dtype=torch.uint8, device=dev)
y = torch.empty_like(x)
pats = {"0x00": lambda: x.fill_(0), "0x03": lambda: x.fill_(3), "0x55": lambda: x.fill_(0x55),
        "0xff": lambda: x.fill_(0xff), "random": lambda: x.copy_(torch.randint(0, 256, (n,), dtype=torch.uint8, device=dev))}
for rep in range(2):
    for name, f in pats.items():
        f()
        t = bench.time_device(torch, lambda: execute_device(p, x, out=y), 15, 3, fl, st)
        tc = bench.time_device(torch, lambda: y.copy_(x), 15, 3, fl, st)
        print(f"{name:7s}: permute {sorted(t)[7]*1e3:6.1f} us   copy_ {sorted(tc)[7]*1e3:6.1f} us", flush=True)
