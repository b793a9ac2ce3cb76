"""e2e (host buffers) timing of a config for several host-pipeline chunk counts."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_03686_b200 as vp  # noqa: E402
from paper_2506_03686_b200.workloads import CONFIGS  # noqa: E402

wl = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg5"]
n = wl.numel * wl.elem_bytes
h_in = torch.randint(0, 255, (n,), dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
for chunks in ["1", "2", "4", "8", "16", "32", "64"]:
    os.environ["VPG_HOST_CHUNKS"] = chunks
    vp.program_cache_clear()
    prog = vp.build_program(vp.TensorLayout.from_shape(wl.shape, wl.elem_bytes), vp.from_numpy_convention(wl.axes))
    best = 1e9
    for _ in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        vp.execute(prog, h_in, out=h_out)
        best = min(best, time.perf_counter() - t0)
    print(f"chunks<={chunks} (used {prog.metadata['host_chunks']}): {best*1e3:.1f} ms  "
          f"{wl.algorithmic_bytes/best/1e9:.1f} GB/s", flush=True)
