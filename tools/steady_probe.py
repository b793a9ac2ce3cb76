"""Steady-state (back-to-back, rotating buffers > 3xL2, PDL) and flushed
single-launch times of the BASELINE configs with the bench's protocol;
optional config list on the command line."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_03686_b200 as vp  # noqa: E402
from paper_2506_03686_b200.api import execute_device  # noqa: E402
from paper_2506_03686_b200.workloads import CONFIGS  # noqa: E402

dev = torch.device("cuda", 0)
fl = bench.Flusher(torch, dev)
st = torch.cuda.current_stream()
class _WL:
    """Ad-hoc workload "d0,d1,...:a0,a1,...:elem" (numpy axes convention)."""

    def __init__(self, spec):
        sh, ax, e = spec.split(":")
        self.shape = tuple(int(v) for v in sh.split(","))
        self.axes = tuple(int(v) for v in ax.split(","))
        self.elem_bytes = int(e)
        self.numel = 1
        for d in self.shape:
            self.numel *= d
        self.algorithmic_bytes = 2 * self.numel * self.elem_bytes


for k in sys.argv[1:] or ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"]:
    wl = CONFIGS[k] if k in CONFIGS else _WL(k)
    n = wl.numel * wl.elem_bytes
    nb = bench.steady_buffers(fl.l2, n)
    xs = [torch.randint(0, 255, (n,), dtype=torch.uint8, device=dev) for _ in range(nb)]
    ys = [torch.empty_like(x) for x in xs]
    prog = vp.build_program(vp.TensorLayout.from_shape(wl.shape, wl.elem_bytes), vp.from_numpy_convention(wl.axes))
    single = bench.time_device(torch, lambda: execute_device(prog, xs[0], out=ys[0]), 20, 3, fl, st)
    s_med = sorted(single)[len(single) // 2] * 1e3
    reps = max(3, min(50, int(4e9 // (nb * 2 * n))))
    ss = [bench.time_steady(torch, lambda i: execute_device(prog, xs[i], out=ys[i]), nb, reps, st) * 1e3
          for _ in range(3)]
    b = wl.algorithmic_bytes
    print(f"{k}: flushed {s_med:7.2f} us ({b / s_med / 1e3:5.0f} GB/s) | steady {min(ss):7.2f}-{max(ss):7.2f} us "
          f"({b / min(ss) / 1e3:5.0f} GB/s) [{nb} buffers] {prog.kernel} {prog.metadata.get('src_run')}x"
          f"{prog.metadata.get('dst_run')}", flush=True)
    del xs, ys
    torch.cuda.empty_cache()
