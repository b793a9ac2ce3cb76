"""How much of a flushed single-launch event time is host enqueue latency?

Protocol A (bench.py r1): per step flush(); ev_a; launch; ev_b -- the host
enqueues each step while the GPU runs the previous one, so if the host is
slower than the flush the GPU idles between ev_a and the kernel.
Protocol B: a ~20 ms spin kernel (torch.cuda._sleep) is enqueued first and
every step queues behind it, so the GPU never waits on the host inside a
timed region (nvbench's blocking-kernel method).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_03686_b200 as vp  # noqa: E402
from paper_2506_03686_b200.api import execute_device  # noqa: E402
from paper_2506_03686_b200.workloads import CONFIGS  # noqa: E402

dev = torch.device("cuda", 0)
st = torch.cuda.current_stream()
fl = bench.Flusher(torch, dev)


def prot_a(launch, n=30):
    t = bench.time_device(torch, launch, n, 3, fl, st)
    t = sorted(v * 1e3 for v in t)
    return round(t[len(t) // 2], 2), round(t[0], 2)


def prot_b(launch, n=30):
    for _ in range(3):
        fl()
        launch()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    torch.cuda._sleep(40_000_000)          # ~20 ms at 1.9 GHz
    for a, b in evs:
        fl()
        a.record(st)
        launch()
        b.record(st)
    torch.cuda.synchronize()
    t = sorted(a.elapsed_time(b) * 1e3 for a, b in evs)
    return round(t[len(t) // 2], 2), round(t[0], 2)


one = torch.zeros(1, dtype=torch.int32, device=dev)
print("1-elem fill  A", prot_a(lambda: one.fill_(1)), " B", prot_b(lambda: one.fill_(1)), flush=True)
for k in ("cfg1", "cfg2", "cfg3"):
    wl = CONFIGS[k]
    n = wl.numel * wl.elem_bytes
    x = torch.randint(0, 255, (n,), dtype=torch.uint8, device=dev)
    y = torch.empty_like(x)
    p = vp.build_program(vp.TensorLayout.from_shape(wl.shape, wl.elem_bytes), vp.from_numpy_convention(wl.axes))
    run = lambda: execute_device(p, x, out=y, stream=st)  # noqa: E731
    cp = lambda: y.copy_(x)  # noqa: E731
    ideal = wl.algorithmic_bytes / 6555.2e3
    print(k, f"ideal {ideal:.2f} us", "perm A", prot_a(run), "B", prot_b(run), "| copy_ A", prot_a(cp), "B",
          prot_b(cp), flush=True)
