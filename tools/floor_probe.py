"""Launch-floor probe: event time of tiny launches of each kernel class."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2506_03686_b200 import TensorLayout, build_program, from_numpy_convention  # noqa: E402
from paper_2506_03686_b200.api import execute_device  # noqa: E402

dev = torch.device("cuda", 0)
fl = bench.Flusher(torch, dev)
st = torch.cuda.current_stream()
x = torch.zeros(1 << 16, dtype=torch.int32, device=dev)
y = torch.empty_like(x)
one = torch.zeros(1, dtype=torch.int32, device=dev)


def med(f):
    t = bench.time_device(torch, f, 30, 5, fl, st)
    return sorted(t)[15] * 1e3


print(f"torch fill_(1 elem): {med(lambda: one.fill_(1)):.2f} us")
for name, shape, axes, force in [("copy", (4096,), (0,), None), ("gather", (32, 32), (1, 0), "gather"),
                                 ("tile 4096", (64, 64), (1, 0), "tile"), ("tile 65536", (256, 256), (1, 0), "tile"),
                                 ("rows", (8, 2, 512), (1, 0, 2), None)]:
    prog = build_program(TensorLayout.from_shape(shape, 4), from_numpy_convention(axes), force=force)
    n = prog.num_elements
    xi, yi = x[:n], y[:n]
    print(f"{name} [{prog.kernel}]: {med(lambda: execute_device(prog, xi, out=yi)):.2f} us")
# host-side launch cost (no GPU wait): 1000 launches wall time
import time  # noqa: E402
prog = build_program(TensorLayout.from_shape((64, 64), 4), from_numpy_convention((1, 0)), force="tile")
xi, yi = x[:4096], y[:4096]
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(1000):
    execute_device(prog, xi, out=yi)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"host launch cost per execute_device: {(t1-t0)*1e3:.2f} us")
