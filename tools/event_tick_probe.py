"""Resolution of CUDA-event timing on this GPU: event pairs around spin
kernels of increasing length (torch.cuda._sleep), the distinct elapsed
values seen and their spacing.  A coarse event clock quantises every
single-launch measurement (the bench's flushed protocol times one launch
per event pair, so small configs are reported as means over many launches)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

st = torch.cuda.current_stream()
torch.cuda._sleep(1000)
torch.cuda.synchronize()
allv = []
for cycles in (0, 2000, 5000, 10000, 20000, 40000):
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(200)]
    for a, b in evs:
        a.record(st)
        if cycles:
            torch.cuda._sleep(cycles)
        b.record(st)
    torch.cuda.synchronize()
    v = np.array([a.elapsed_time(b) * 1e3 for a, b in evs])
    allv.append(v)
    u, c = np.unique(np.round(v, 3), return_counts=True)
    print(f"sleep {cycles:6d} cycles: mean {v.mean():7.3f} us  distinct values (us: count) "
          + ", ".join(f"{x:.3f}: {n}" for x, n in zip(u[:8], c[:8])), flush=True)
vals = np.unique(np.round(np.concatenate(allv), 3))
d = np.diff(vals)
print(f"smallest nonzero spacing between distinct elapsed values: {d[d > 0].min() if d.size else 0:.3f} us; "
      f"all values multiples of 2.048 us: {bool(np.all(np.abs(vals / 2.048 - np.round(vals / 2.048)) < 1e-3))}")

# the same pairs after the bench's L2 flush (bench.Flusher: a 2xL2 write and
# a 2xL2 read): the start event waits for the flush kernel to finish
import bench  # noqa: E402

fl = bench.Flusher(torch, torch.device("cuda", 0))
print("-- after an L2 flush (bench protocol)")
allf = []
for cycles in (0, 2000, 5000, 10000, 15000, 20000, 25000, 40000):
    res = []
    for _ in range(40):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fl()
        a.record(st)
        if cycles:
            torch.cuda._sleep(cycles)
        b.record(st)
        res.append((a, b))
    torch.cuda.synchronize()
    v = np.array([a.elapsed_time(b) * 1e3 for a, b in res])
    allf.append(v)
    u, c = np.unique(np.round(v, 3), return_counts=True)
    ticks = np.abs(v / 2.048 - np.round(v / 2.048)) < 0.01
    print(f"sleep {cycles:6d} cycles: mean {v.mean():7.3f} us  on a 2.048 us multiple: {ticks.mean() * 100:5.1f}%  "
          + ", ".join(f"{x:.3f}: {n}" for x, n in zip(u[:6], c[:6])), flush=True)
