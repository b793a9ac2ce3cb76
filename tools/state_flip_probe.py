"""Within ONE process: does the cfg5 kernel time change after a 2 GiB H2D
copy, a D2D copy, or an autotune?  (Interleaved events.)"""
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
n = wl.numel * wl.elem_bytes
lay, pm = vp.TensorLayout.from_shape(wl.shape, 8), vp.from_numpy_convention(wl.axes)
p = vp.build_program(lay, pm)
fl = bench.Flusher(torch, dev)
st = torch.cuda.current_stream()
x = torch.randint(0, 255, (n,), dtype=torch.uint8, device=dev)
y = torch.empty_like(x)
scratch = torch.empty_like(x)
host = torch.empty(n, dtype=torch.uint8, pin_memory=True)


def med():
    t = bench.time_device(torch, lambda: execute_device(p, x, out=y), 15, 3, fl, st)
    return round(sorted(t)[7] * 1e3, 1)


print("start            ", med(), med(), flush=True)
scratch.copy_(host)
torch.cuda.synchronize()
print("after H2D scratch", med(), med(), flush=True)
x.copy_(host)
torch.cuda.synchronize()
print("after H2D into x ", med(), med(), flush=True)
x.copy_(torch.randint(0, 255, (n,), dtype=torch.uint8, device=dev))
print("after x rewritten", med(), med(), flush=True)
scratch.copy_(x)
print("after D2D        ", med(), med(), flush=True)
vp.autotune(lay, pm, src=x, dst=y)
print("after autotune   ", med(), med(), flush=True)
