"""Is a plan slower after autotune ran in the same process?"""
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
lay, pm = vp.TensorLayout.from_shape(wl.shape, wl.elem_bytes), vp.from_numpy_convention(wl.axes)
c1 = vp.build_program(lay, pm, candidate=1)
x = torch.randint(0, 255, (n,), dtype=torch.uint8, device=dev)
y = torch.empty_like(x)


def med():
    t = bench.time_device(torch, lambda: execute_device(c1, x, out=y), 15, 3, fl, st)
    return round(sorted(t)[7] * 1e3, 1)


print("before autotune:", med(), med())
vp.autotune(lay, pm)
print("after autotune :", med(), med())
torch.cuda.empty_cache()
print("after empty_cache:", med())
