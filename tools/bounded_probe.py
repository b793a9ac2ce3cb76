"""Host-path throughput through bounded device scratch (cfg5, pinned)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_03686_b200 as vp  # noqa: E402
from paper_2506_03686_b200.workloads import CONFIGS  # noqa: E402

wl = CONFIGS["cfg5"]
n = wl.numel * wl.elem_bytes
h_in = torch.randint(0, 255, (n,), dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
prog = vp.build_program(vp.TensorLayout.from_shape(wl.shape, wl.elem_bytes), vp.from_numpy_convention(wl.axes))
for mib in (4096, 1024, 256, 64):
    kw = {} if mib >= 4096 else {"max_device_bytes": mib << 20}
    vp.execute(prog, h_in, out=h_out, **kw)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        vp.execute(prog, h_in, out=h_out, **kw)
    dt = (time.perf_counter() - t0) / 3
    print(f"scratch {'full' if not kw else str(mib) + ' MiB':>9}: {wl.algorithmic_bytes / dt / 1e9:6.1f} GB/s", flush=True)
