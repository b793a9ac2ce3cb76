"""Back-to-back launches over rotating buffers (inputs and outputs > L2 in
total, no flush): steady-state per-launch time vs the flushed single launch."""
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
for k in ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"]:
    wl = CONFIGS[k]
    n = wl.numel * wl.elem_bytes
    nb = max(2, min(16, (1 << 30) // n))
    xs = [torch.randint(0, 255, (n,), dtype=torch.uint8, device=dev) for _ in range(nb)]
    ys = [torch.empty_like(x) for x in xs]
    prog = vp.build_program(vp.TensorLayout.from_shape(wl.shape, wl.elem_bytes), vp.from_numpy_convention(wl.axes))
    single = bench.time_device(torch, lambda: execute_device(prog, xs[0], out=ys[0]), 10, 3, fl, st)
    s_med = sorted(single)[len(single) // 2] * 1e3
    reps = 3
    for i in range(nb):
        execute_device(prog, xs[i], out=ys[i])
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(st)
    for _ in range(reps):
        for i in range(nb):
            execute_device(prog, xs[i], out=ys[i])
    b.record(st)
    torch.cuda.synchronize()
    per = a.elapsed_time(b) * 1e3 / (reps * nb)
    tc = []
    a.record(st)
    for _ in range(reps):
        for i in range(nb):
            ys[i].copy_(xs[i])
    b.record(st)
    torch.cuda.synchronize()
    cper = a.elapsed_time(b) * 1e3 / (reps * nb)
    print(f"{k}: flushed single {s_med:7.1f} us ({wl.algorithmic_bytes/s_med/1e3:5.0f} GB/s) | back-to-back "
          f"{per:7.1f} us ({wl.algorithmic_bytes/per/1e3:5.0f} GB/s) | copy_ back-to-back {cper:7.1f} us "
          f"({wl.algorithmic_bytes/cper/1e3:5.0f} GB/s) [{nb} buffers]", flush=True)
    del xs, ys
    torch.cuda.empty_cache()
