"""Per-config timing probe: flushed single launches vs back-to-back launches,
plus an empty-work launch floor.  Prints one line per config."""
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
cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else sorted(CONFIGS)
# floor: smallest possible launch through the same API
tiny = build_program(TensorLayout((2048, 2)), from_numpy_convention((1, 0)), force="tile")
xt = torch.zeros(4096, dtype=torch.int32, device=dev)
yt = torch.empty_like(xt)
t = bench.time_device(torch, lambda: execute_device(tiny, xt, out=yt), 20, 5, fl, st)
print(f"floor (4096-elem tile launch): median {sorted(t)[10]*1e3:.2f} us", flush=True)
for k in cfgs:
    wl = CONFIGS[k]
    prog = build_program(TensorLayout.from_shape(wl.shape, wl.elem_bytes), from_numpy_convention(wl.axes))
    n = wl.numel * wl.elem_bytes
    x = torch.randint(0, 255, (n,), dtype=torch.uint8, device=dev)
    y = torch.empty_like(x)
    f = lambda: execute_device(prog, x, out=y)  # noqa: E731
    tf = bench.time_device(torch, f, 20, 5, fl, st)
    # back-to-back (no flush), 20 launches inside one event pair
    for _ in range(3):
        f()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(20):
        f()
    b.record(st)
    torch.cuda.synchronize()
    bb = a.elapsed_time(b) / 20
    med = sorted(tf)[10]
    # batched distinct buffers (> 2x L2 in total): event overhead amortised
    nb = max(2, int((4 * fl.l2) // (2 * n)) + 1)
    xs = [torch.randint(0, 255, (n,), dtype=torch.uint8, device=dev) for _ in range(nb)]
    ys = [torch.empty_like(xx) for xx in xs]
    for i in range(nb):
        execute_device(prog, xs[i], out=ys[i])
    fl()
    a2, b2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a2.record(st)
    for i in range(nb):
        execute_device(prog, xs[i], out=ys[i])
    b2.record(st)
    torch.cuda.synchronize()
    bt = a2.elapsed_time(b2) / nb
    del xs, ys
    print(f"{k}: flushed median {med*1e3:.1f} us ({wl.algorithmic_bytes/med/1e6:.0f} GB/s) best {min(tf)*1e3:.1f}; "
          f"back-to-back {bb*1e3:.1f} us; batched-distinct x{nb} {bt*1e3:.1f} us ({wl.algorithmic_bytes/bt/1e6:.0f} GB/s)  [{prog.kernel}]", flush=True)
