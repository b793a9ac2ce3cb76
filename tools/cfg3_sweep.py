"""Planner-knob sweep of one BASELINE config (default cfg3) in the bench's
flushed protocol and the steady protocol: tile budget x pipeline depth x
CTA threads x W mode (VPG_LIN), each plan rebuilt in-process (the knobs are
read at plan creation).  Prints one line per setting, then the best ten by
flushed median.   usage: python tools/cfg3_sweep.py [cfg3] [quick]"""
import itertools
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_03686_b200 as vp  # noqa: E402
from paper_2506_03686_b200.api import execute_device  # noqa: E402
from paper_2506_03686_b200.workloads import CONFIGS  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
quick = len(sys.argv) > 2
wl = CONFIGS[cfg]
dev = torch.device("cuda", 0)
fl = bench.Flusher(torch, dev)
st = torch.cuda.current_stream()
peak = bench._peaks()[0]
n = wl.numel * wl.elem_bytes
x = torch.randint(0, 255, (n,), dtype=torch.uint8, device=dev)
y = torch.empty_like(x)
nb = bench.steady_buffers(fl.l2, n)
xs = [x] + [x.clone() for _ in range(nb - 1)]
ys = [y] + [torch.empty_like(x) for _ in range(nb - 1)]
tdt = {4: torch.int32, 8: torch.int64}[wl.elem_bytes]
KEYS = ("VPG_TILE_BUDGET", "VPG_NBUF", "VPG_THREADS", "VPG_LIN", "VPG_PERSIST")
grid = {
    "VPG_TILE_BUDGET": [None, "16384", "24576", "40960", "49152"],
    "VPG_NBUF": [None, "3", "4"],
    "VPG_THREADS": [None, "384", "512"],
    "VPG_LIN": ["0", "1"],
    "VPG_PERSIST": [None],
}
if quick:
    grid = {"VPG_TILE_BUDGET": [None, "24576"], "VPG_NBUF": [None, "3"], "VPG_THREADS": [None], "VPG_LIN": ["0", "1"],
            "VPG_PERSIST": [None]}
if os.environ.get("SWEEP_GRID"):          # JSON {knob: [values or null]}, missing knobs at default
    grid = {k: [None] for k in KEYS}
    grid.update(json.loads(os.environ["SWEEP_GRID"]))
res = []
for combo in itertools.product(*(grid[k] for k in KEYS)):
    for k, v in zip(KEYS, combo):
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v
    vp.program_cache_clear()
    tag = " ".join(f"{k[4:]}={v}" for k, v in zip(KEYS, combo) if v is not None) or "default"
    try:
        p = vp.build_program(vp.TensorLayout.from_shape(wl.shape, wl.elem_bytes), vp.from_numpy_convention(wl.axes))
        run = lambda: execute_device(p, x, out=y, stream=st)  # noqa: E731
        t = sorted(bench.time_device(torch, run, 31, 3, fl, st))
        med = t[len(t) // 2] * 1e3
        ok = bench.sample_parity(torch, x.view(tdt), y.view(tdt), wl.shape, wl.axes, nsamp=1 << 16)
        reps = max(3, min(50, int(4e9 // (nb * 2 * n))))
        sm = min(bench.time_steady(torch, lambda i: execute_device(p, xs[i], out=ys[i], stream=st), nb, reps, st)
                 for _ in range(2)) * 1e3
    except Exception as e:  # noqa: BLE001
        print(f"{tag}: {type(e).__name__}: {e}", flush=True)
        continue
    meta = p.metadata
    lin = "W lin" in p.text
    line = (f"{tag:48s} T={meta['tile_elems']:6d} {meta['src_run']}x{meta['dst_run']} smem={meta['smem_bytes']} thr={meta['threads']} "
            f"lin={int(lin)} flushed {med:6.2f} us ({wl.algorithmic_bytes / med / 1e3 / peak * 100:5.1f}%) "
            f"steady {sm:6.2f} us ({wl.algorithmic_bytes / sm / 1e3 / peak * 100:5.1f}%) parity {ok}")
    print(line, flush=True)
    res.append((med, line))
for k in KEYS:
    os.environ.pop(k, None)
print("== best by flushed median")
for _, line in sorted(res)[:10]:
    print(line)
