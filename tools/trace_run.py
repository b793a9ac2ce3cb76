"""Trace flushed single launches of BASELINE configs (VPG_TRACE) and
summarise the last one per config (tools/trace_view.py)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
path = "/tmp/vpg_trace.bin"
os.environ["VPG_TRACE"] = path
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_03686_b200 as vp  # noqa: E402
from paper_2506_03686_b200.api import execute_device  # noqa: E402
from paper_2506_03686_b200.workloads import CONFIGS  # noqa: E402
from tools import trace_view  # noqa: E402

dev = torch.device("cuda", 0)
fl = bench.Flusher(torch, dev)
for k in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["cfg2", "cfg3", "cfg1"]):
    if os.path.exists(path):
        os.remove(path)
    wl = CONFIGS[k]
    n = wl.numel * wl.elem_bytes
    x = torch.randint(0, 255, (n,), dtype=torch.uint8, device=dev)
    y = torch.empty_like(x)
    p = vp.build_program(vp.TensorLayout.from_shape(wl.shape, wl.elem_bytes), vp.from_numpy_convention(wl.axes))
    for _ in range(4):
        fl()
        execute_device(p, x, out=y)
    torch.cuda.synchronize()
    print("== flushed", k)
    ls = list(trace_view.launches(path))
    trace_view.summarise(*ls[-1])
    if os.environ.get("TRACE_STEADY"):
        # back to back on rotating buffers (no flush): code and constants warm
        nb = bench.steady_buffers(fl.l2, n)
        xs = [x] + [x.clone() for _ in range(nb - 1)]
        ys = [y] + [torch.empty_like(x) for _ in range(nb - 1)]
        for r in range(2):
            for i in range(nb):
                execute_device(p, xs[i], out=ys[i])
        torch.cuda.synchronize()
        print("== back-to-back", k)
        ls = list(trace_view.launches(path))
        trace_view.summarise(*ls[-1])
        del xs, ys
