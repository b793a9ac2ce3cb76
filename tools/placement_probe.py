"""Does the relative placement of src and dst change the cfg5 kernel time?
One pool, src fixed at its start, dst at a series of offsets."""
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
fl = bench.Flusher(torch, dev)
st = torch.cuda.current_stream()
n = wl.numel * wl.elem_bytes
lay, pm = vp.TensorLayout.from_shape(wl.shape, wl.elem_bytes), vp.from_numpy_convention(wl.axes)
progs = {c: vp.build_program(lay, pm, candidate=c) for c in (0, 1)}
pool = torch.empty(2 * n + (1 << 30), dtype=torch.uint8, device=dev)
print("pool", hex(pool.data_ptr()))
x = pool[:n]
x.copy_(torch.randint(0, 255, (n,), dtype=torch.uint8, device=dev))
MB = 1 << 20
for off in [n, n + 2 * MB, n + 64 * MB, n + 128 * MB, n + 256 * MB, n + 512 * MB, n + 768 * MB, n + 1024 * MB,
            n + 96 * MB, n + 4 * MB]:
    y = pool[off:off + n]
    row = []
    for c in (0, 1):
        t = bench.time_device(torch, lambda: execute_device(progs[c], x, out=y), 12, 3, fl, st)
        row.append(sorted(t)[6] * 1e3)
    print(f"dst offset {(off - n) // MB:5d} MiB past src end: cand0 {row[0]:6.1f} us  cand1 {row[1]:6.1f} us",
          flush=True)
