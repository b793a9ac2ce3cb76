"""Why does bench.py time the same cfg5 plan slower than tools/pick_ab.py?
Same process: the tuned plan on the bench's buffers, with and without the
NVML clock sampler, and on fresh buffers."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_03686_b200 as vp  # noqa: E402
from paper_2506_03686_b200.api import execute_device  # noqa: E402
from paper_2506_03686_b200.workloads import CONFIGS, make_input  # noqa: E402

wl = CONFIGS["cfg5"]
dev = torch.device("cuda", 0)
fl = bench.Flusher(torch, dev)
st = torch.cuda.current_stream()
n = wl.numel * wl.elem_bytes
lay, pm = vp.TensorLayout.from_shape(wl.shape, wl.elem_bytes), vp.from_numpy_convention(wl.axes)
prog = vp.build_program(lay, pm, tune=True)
print("tuned", prog.metadata["src_run"], prog.metadata["dst_run"], prog.metadata.get("tuned_ms"))
host_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
host_in.numpy()[:] = make_input(wl, threads=16).reshape(-1).view("u1")
xd = host_in.to(dev)
yd = torch.empty_like(xd)


def med(x, y):
    t = bench.time_device(torch, lambda: execute_device(prog, x, out=y), 20, 5, fl, st)
    return sorted(t)[10] * 1e3


print("bench buffers, no sampler  :", round(med(xd, yd), 1))
with bench.ClockSampler(0):
    print("bench buffers, sampler on  :", round(med(xd, yd), 1))
print("bench buffers, no sampler  :", round(med(xd, yd), 1))
x2 = torch.empty_like(xd).copy_(xd)
y2 = torch.empty_like(xd)
print("fresh buffers              :", round(med(x2, y2), 1))
print("bench x, fresh y           :", round(med(xd, y2), 1))
print("fresh x, bench y           :", round(med(x2, yd), 1))
print("ptrs", hex(xd.data_ptr()), hex(yd.data_ptr()), hex(x2.data_ptr()), hex(y2.data_ptr()))
