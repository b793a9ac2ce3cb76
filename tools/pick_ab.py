"""Interleaved A/B of tile candidates (flushed single launches, median of 15)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_03686_b200 as vp  # noqa: E402
from paper_2506_03686_b200.api import execute_device  # noqa: E402
from paper_2506_03686_b200.workloads import CONFIGS  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
picks = [int(a) for a in (sys.argv[2] if len(sys.argv) > 2 else "0,1").split(",")]
wl = CONFIGS[cfg]
dev = torch.device("cuda", 0)
fl = bench.Flusher(torch, dev)
st = torch.cuda.current_stream()
n = wl.numel * wl.elem_bytes
x = torch.randint(0, 255, (n,), dtype=torch.uint8, device=dev)
y = torch.empty_like(x)
lay, pm = vp.TensorLayout.from_shape(wl.shape, wl.elem_bytes), vp.from_numpy_convention(wl.axes)
progs = {c: vp.build_program(lay, pm, candidate=c) for c in picks}
res = {c: [] for c in picks}
for rep in range(6):
    for c in picks:
        t = bench.time_device(torch, lambda: execute_device(progs[c], x, out=y), 15, 3, fl, st)
        res[c].append(sorted(t)[7] * 1e3)
for c in picks:
    m = progs[c].metadata
    ts = res[c]
    print(f"{cfg} cand {c} ({m['src_run']}x{m['dst_run']}, pitch {m['smem_pitch']}): "
          f"{[round(v, 1) for v in ts]} mean {sum(ts)/len(ts):.1f} us", flush=True)
