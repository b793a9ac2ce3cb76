"""Streaming (non-blocking) host-path throughput vs host-pipeline chunk count."""
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
outs = [torch.empty(n, dtype=torch.uint8).pin_memory() for _ in range(2)]
for chunks in ["1", "2", "4", "8", "16"]:
    os.environ["VPG_HOST_CHUNKS"] = chunks
    vp.program_cache_clear()
    vp.release_scratch()
    prog = vp.build_program(vp.TensorLayout.from_shape(wl.shape, wl.elem_bytes), vp.from_numpy_convention(wl.axes))
    for s in range(3):
        vp.execute(prog, h_in, out=outs[s % 2], blocking=False)
    torch.cuda.synchronize()
    K = 8
    t0 = time.perf_counter()
    for s in range(K):
        vp.execute(prog, h_in, out=outs[s % 2], blocking=False)
    torch.cuda.current_stream().synchronize()
    dt = (time.perf_counter() - t0) / K
    print(f"chunks<={chunks} (used {prog.metadata['host_chunks']}): {dt*1e3:.1f} ms/step "
          f"{wl.algorithmic_bytes/dt/1e9:.1f} GB/s", flush=True)
