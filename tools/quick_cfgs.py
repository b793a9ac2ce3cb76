"""Flushed-median and steady-state us per BASELINE config (bench.py protocols),
for quick A/B of kernel changes.  usage: python tools/quick_cfgs.py [cfg1,cfg3,...]
Env knobs (VPG_*) apply to every plan of the run."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_03686_b200 as vp  # noqa: E402
from paper_2506_03686_b200.api import execute_device  # noqa: E402
from paper_2506_03686_b200.workloads import CONFIGS  # noqa: E402

cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"]
steps = int(os.environ.get("QC_STEPS", "30"))
dev = torch.device("cuda", 0)
fl = bench.Flusher(torch, dev)
st = torch.cuda.current_stream()
peak = bench._peaks()[0]
for k in cfgs:
    wl = CONFIGS[k]
    n = wl.numel * wl.elem_bytes
    x = torch.randint(0, 255, (n,), dtype=torch.uint8, device=dev)
    y = torch.empty_like(x)
    p = vp.build_program(vp.TensorLayout.from_shape(wl.shape, wl.elem_bytes), vp.from_numpy_convention(wl.axes))
    run = lambda: execute_device(p, x, out=y, stream=st)  # noqa: E731
    t = sorted(bench.time_device(torch, run, steps, 3, fl, st))
    med = t[len(t) // 2] * 1e3
    mean = sum(t) / len(t) * 1e3
    tdt = {4: torch.int32, 8: torch.int64}[wl.elem_bytes]
    ok = bench.sample_parity(torch, x.view(tdt), y.view(tdt), wl.shape, wl.axes, nsamp=1 << 18)
    nb = bench.steady_buffers(fl.l2, n)
    xs = [x] + [x.clone() for _ in range(nb - 1)]
    ys = [y] + [torch.empty_like(x) for _ in range(nb - 1)]
    reps = max(3, min(50, int(4e9 // (nb * 2 * n))))
    sm = min(bench.time_steady(torch, lambda i: execute_device(p, xs[i], out=ys[i], stream=st), nb, reps, st)
             for _ in range(2)) * 1e3
    b = wl.algorithmic_bytes
    print(f"{k}: flushed median {med:7.2f} us mean {mean:7.2f} ({b / mean / 1e3 / peak * 100:5.1f}% mean) "
          f"steady {sm:7.2f} us ({b / sm / 1e3 / peak * 100:5.1f}%)  parity {ok}  kernel {p.kernel}", flush=True)
    del xs, ys, x, y
    torch.cuda.empty_cache()
