"""Sweep planner knobs (VPG_* env overrides) over configs; flushed median us
(SWEEP_MODE=steady: best steady-state per-launch us)."""
import itertools
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2506_03686_b200 import TensorLayout, build_program, from_numpy_convention, program_cache_clear  # noqa: E402
from paper_2506_03686_b200.api import execute_device  # noqa: E402
from paper_2506_03686_b200.workloads import CONFIGS  # noqa: E402

cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["cfg1", "cfg2", "cfg3"]
import json  # noqa: E402
grid = json.loads(os.environ.get("SWEEP_GRID", "{}")) or {
    "VPG_TILE_BUDGET": ["16384", "32768", "49152"],
    "VPG_CTA_SMEM": ["70000", "110000", "150000", "220000"],
}
dev = torch.device("cuda", 0)
fl = bench.Flusher(torch, dev)
st = torch.cuda.current_stream()
for k in cfgs:
    wl = CONFIGS[k]
    n = wl.numel * wl.elem_bytes
    steady = os.environ.get("SWEEP_MODE") == "steady"     # back-to-back over rotating buffers (PDL)
    nb = bench.steady_buffers(fl.l2, n) if steady else 1
    xs = [torch.randint(0, 255, (n,), dtype=torch.uint8, device=dev) for _ in range(nb)]
    ys = [torch.empty_like(x) for x in xs]
    x, y = xs[0], ys[0]
    res = []
    for vals in itertools.product(*grid.values()):
        env = dict(zip(grid.keys(), vals))
        os.environ.update(env)
        program_cache_clear()
        prog = build_program(TensorLayout.from_shape(wl.shape, wl.elem_bytes), from_numpy_convention(wl.axes))
        if steady:
            med = min(bench.time_steady(torch, lambda i: execute_device(prog, xs[i], out=ys[i]), nb, 10, st)
                      for _ in range(3)) * 1e3
        else:
            t = bench.time_device(torch, lambda: execute_device(prog, x, out=y), 15, 3, fl, st)
            med = sorted(t)[len(t) // 2] * 1e3
        res.append((med, env, prog.metadata["tile_elems"], prog.metadata["smem_bytes"]))
    res.sort(key=lambda r: r[0])
    for med, env, te, sm in res[:6]:
        print(f"{k} {med:7.1f} us {wl.algorithmic_bytes/med/1e3:7.0f} GB/s tile={te} smem={sm} {env}", flush=True)
    print(f"{k} worst {res[-1][0]:.1f} us", flush=True)
