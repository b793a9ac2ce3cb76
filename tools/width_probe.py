"""Same-byte 2-D transposes at 4/8/16-byte words (flushed, event-timed):
how much the W phase's per-word stores cost."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_03686_b200 as vp  # noqa: E402
from paper_2506_03686_b200.api import execute_device  # noqa: E402

dev = torch.device("cuda", 0)
fl = bench.Flusher(torch, dev)
st = torch.cuda.current_stream()
for rows, cols, E in [(4096, 4096, 4), (4096, 2048, 8), (4096, 1024, 16), (2048, 4096, 8), (1024, 4096, 16),
                      (8192, 8192, 4), (8192, 4096, 8), (8192, 2048, 16)]:
    nbytes = rows * cols * E
    x = torch.randint(0, 255, (nbytes,), dtype=torch.uint8, device=dev)
    y = torch.empty_like(x)
    prog = vp.build_program(vp.TensorLayout.from_shape((rows, cols), E), vp.from_numpy_convention((1, 0)))
    t = bench.time_device(torch, lambda: execute_device(prog, x, out=y), 15, 3, fl, st)
    med = sorted(t)[len(t) // 2] * 1e3
    m = prog.metadata
    print(f"{rows}x{cols} E={E:2d}: {med:7.1f} us {2*nbytes/med/1e3:7.0f} GB/s  tile {m['src_run']}x{m['dst_run']} "
          f"vec {m['vec_elems']}", flush=True)
