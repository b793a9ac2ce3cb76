"""Does the data pattern change kernel time?  cfg5 plan, inputs of zeros,
random bytes and the bench's seeded normal complex64 values."""
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
xs = {
    "zeros": torch.zeros(n, dtype=torch.uint8, device=dev),
    "random bytes": torch.randint(0, 255, (n,), dtype=torch.uint8, device=dev),
    "bench normal c64": torch.from_numpy(make_input(wl, threads=16).reshape(-1).view(np.uint8)).to(dev),
}
y = torch.empty(n, dtype=torch.uint8, device=dev)
lay, pm = vp.TensorLayout.from_shape(wl.shape, wl.elem_bytes), vp.from_numpy_convention(wl.axes)
for c in (0, 1):
    prog = vp.build_program(lay, pm, candidate=c)
    for rep in range(2):
        for name, x in xs.items():
            t = bench.time_device(torch, lambda: execute_device(prog, x, out=y), 15, 3, fl, st)
            print(f"cand {c} {name:18s}: {sorted(t)[7] * 1e3:7.1f} us", flush=True)
    for name, x in xs.items():
        t = bench.time_device(torch, lambda: y.copy_(x), 15, 3, fl, st)
        print(f"copy_  {name:18s}: {sorted(t)[7] * 1e3:7.1f} us", flush=True)
