"""Distribution of 40 flushed single launches of cfg2 and of a 1-element
kernel (event resolution and the bimodal launch timing of small kernels)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch, bench
import paper_2506_03686_b200 as vp
from paper_2506_03686_b200.api import execute_device
from paper_2506_03686_b200.workloads import CONFIGS
dev = torch.device("cuda", 0); fl = bench.Flusher(torch, dev); st = torch.cuda.current_stream()
wl = CONFIGS["cfg2"]; n = wl.numel * 4
x = torch.randint(0, 255, (n,), dtype=torch.uint8, device=dev); y = torch.empty_like(x)
p = vp.build_program(vp.TensorLayout.from_shape(wl.shape, 4), vp.from_numpy_convention(wl.axes))
t = bench.time_device(torch, lambda: execute_device(p, x, out=y), 40, 3, fl, st)
print(sorted(round(v * 1e3, 3) for v in t))
one = torch.zeros(1, device=dev)
t = bench.time_device(torch, lambda: one.fill_(1), 40, 3, fl, st)
print(sorted(round(v * 1e3, 3) for v in t))
# the same with an L2 flush done by one of our own tile kernels (a 512 MiB
# transpose: same shared-memory configuration as the timed kernel)
big = torch.empty(128 << 20, dtype=torch.float32, device=dev)
bigo = torch.empty_like(big)
pf = vp.build_program(vp.TensorLayout.from_shape((8192, 16384), 4), vp.from_numpy_convention((1, 0)))
own_flush = lambda: execute_device(pf, big, out=bigo)  # noqa: E731
t = bench.time_device(torch, lambda: execute_device(p, x, out=y), 40, 3, own_flush, st)
print("own-kernel flush:", sorted(round(v * 1e3, 3) for v in t))
