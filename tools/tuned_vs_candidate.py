"""The autotuned cfg5 program vs the same candidate built directly (same object, same timing)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch, bench
import paper_2506_03686_b200 as vp
from paper_2506_03686_b200.api import execute_device
from paper_2506_03686_b200.workloads import CONFIGS
wl = CONFIGS["cfg5"]
lay, pm = vp.TensorLayout.from_shape(wl.shape, wl.elem_bytes), vp.from_numpy_convention(wl.axes)
tuned = vp.build_program(lay, pm, tune=True)
c1 = vp.build_program(lay, pm, candidate=1)
print("same object:", tuned is c1)
print("TUNED\n", tuned.text)
print("C1\n", c1.text)
dev = torch.device("cuda", 0); fl = bench.Flusher(torch, dev); st = torch.cuda.current_stream()
n = wl.numel * 8
x = torch.randint(0, 255, (n,), dtype=torch.uint8, device=dev); y = torch.empty_like(x)
for rep in range(3):
    for name, p in (("tuned", tuned), ("c1", c1)):
        t = bench.time_device(torch, lambda: execute_device(p, x, out=y), 15, 3, fl, st)
        print(name, round(sorted(t)[7] * 1e3, 1), p.jit_state)
