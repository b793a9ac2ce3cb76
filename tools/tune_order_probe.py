"""Process-order probe: time candidate 1 of cfg5 when built directly (A),
as the autotune winner (B), or rebuilt after an autotune (C)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_03686_b200 as vp  # noqa: E402
from paper_2506_03686_b200.api import execute_device  # noqa: E402
from paper_2506_03686_b200.workloads import CONFIGS  # noqa: E402

mode = sys.argv[1]
pre = len(sys.argv) > 2 and sys.argv[2] == "pre"     # allocate flush/x/y before the prelude
wl = CONFIGS["cfg5"]
dev = torch.device("cuda", 0)
n = wl.numel * wl.elem_bytes
lay, pm = vp.TensorLayout.from_shape(wl.shape, wl.elem_bytes), vp.from_numpy_convention(wl.axes)
if pre:
    fl = bench.Flusher(torch, dev)
    x = torch.randint(0, 255, (n,), dtype=torch.uint8, device=dev)
    y = torch.empty_like(x)
if mode == "A":
    p = vp.build_program(lay, pm, candidate=1)
elif mode == "B":
    p = vp.autotune(lay, pm)
elif mode.startswith("T"):  # autotune with k candidates ("T4")
    p = vp.autotune(lay, pm, candidates=int(mode[1:]))
elif mode in ("Z", "Zi", "Zs"):  # autotune's timing helper on c1 alone (Zi: initialised src, Zs: no per-launch sync)
    from paper_2506_03686_b200.api import _time_program
    p = vp.build_program(lay, pm, candidate=1)
    sa = torch.empty(n, dtype=torch.uint8, device=dev)
    if mode == "Zi":
        sa.fill_(7)
    da = torch.empty(n, dtype=torch.uint8, device=dev)
    flb = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    if mode == "Zs":
        for _ in range(7):
            flb.zero_()
            execute_device(p, sa, out=da)
        torch.cuda.synchronize()
    else:
        _time_program(torch, p, sa, da, flb, 5)
    del sa, da, flb
elif mode in ("S1", "S2"):   # flush buffers carved from a freed 2 GiB block (S1), or x/y from it (S2)
    p = vp.build_program(lay, pm, candidate=1)
    big = torch.empty(n, dtype=torch.uint8, device=dev)
    del big
    if mode == "S1":
        fl = bench.Flusher(torch, dev)
        x = torch.randint(0, 255, (n,), dtype=torch.uint8, device=dev)
        y = torch.empty_like(x)
        pre = True
elif mode in ("Q", "Q2"):   # bench-like input: pinned host buffer copied to the device (Q2: + NVML sampler)
    p = vp.build_program(lay, pm, candidate=1)
    host_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    host_in.fill_(3)
    fl = bench.Flusher(torch, dev)
    x = host_in.to(dev)
    y = torch.empty_like(x)
    pre = True
    if mode == "Q2":
        _clk = bench.ClockSampler(0)
        _clk.__enter__()
elif mode in ("Q3", "Q4", "Q5"):
    # Q3: 2 GiB pinned host allocation, device input written by a kernel
    # Q4: pageable host buffer copied in;  Q5: device input written by a kernel, then a 2 GiB D2D copy into it
    p = vp.build_program(lay, pm, candidate=1)
    fl = bench.Flusher(torch, dev)
    if mode == "Q3":
        host_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        host_in.fill_(3)
        x = torch.randint(0, 255, (n,), dtype=torch.uint8, device=dev)
    elif mode == "Q4":
        host_in = torch.empty(n, dtype=torch.uint8)
        host_in.fill_(3)
        x = host_in.to(dev)
    else:
        x = torch.randint(0, 255, (n,), dtype=torch.uint8, device=dev)
        x.copy_(torch.randint(0, 255, (n,), dtype=torch.uint8, device=dev))
    y = torch.empty_like(x)
    pre = True
elif mode == "U":          # autotune on the bench buffers
    assert pre
    p = vp.autotune(lay, pm, src=x, dst=y)
elif mode in ("W1", "W0"):  # one launch of candidate 1 / 0 on the bench buffers, then autotune
    assert pre
    execute_device(vp.build_program(lay, pm, candidate=int(mode[1])), x, out=y)
    torch.cuda.synchronize()
    p = vp.autotune(lay, pm)
elif mode == "C":
    vp.autotune(lay, pm)
    vp.program_cache_clear()
    p = vp.build_program(lay, pm, candidate=1)
elif mode == "D":          # autotune, then return its scratch to the driver
    p = vp.autotune(lay, pm)
    torch.cuda.empty_cache()
elif mode in ("F", "G"):  # launch another candidate's kernel first (F: 0, G: 3)
    other = vp.build_program(lay, pm, candidate=0 if mode == "F" else 3)
    p = vp.build_program(lay, pm, candidate=1)
    xa = torch.empty(n, dtype=torch.uint8, device=dev)
    ya = torch.empty(n, dtype=torch.uint8, device=dev)
    for _ in range(3):
        execute_device(other, xa, out=ya)
    torch.cuda.synchronize()
    del xa, ya
elif mode == "H":          # as much traffic as an autotune, with the same kernel
    p = vp.build_program(lay, pm, candidate=1)
    xa = torch.empty(n, dtype=torch.uint8, device=dev)
    ya = torch.empty(n, dtype=torch.uint8, device=dev)
    for _ in range(70):
        execute_device(p, xa, out=ya)
    torch.cuda.synchronize()
    del xa, ya
elif mode in ("J", "K"):   # as H, then idle 2 s (J) or 10 s (K) before timing
    import time
    p = vp.build_program(lay, pm, candidate=1)
    xa = torch.empty(n, dtype=torch.uint8, device=dev)
    ya = torch.empty(n, dtype=torch.uint8, device=dev)
    for _ in range(70):
        execute_device(p, xa, out=ya)
    torch.cuda.synchronize()
    del xa, ya
    time.sleep(2 if mode == "J" else 10)
elif mode == "I":          # autotune with a single candidate
    p = vp.autotune(lay, pm, candidates=1)
    p = vp.build_program(lay, pm, candidate=1)
elif mode.startswith("P"):  # 7 launches of candidate k first ("P7")
    other = vp.build_program(lay, pm, candidate=int(mode[1:]))
    p = vp.build_program(lay, pm, candidate=1)
    xa = torch.empty(n, dtype=torch.uint8, device=dev)
    ya = torch.empty(n, dtype=torch.uint8, device=dev)
    for _ in range(7):
        execute_device(other, xa, out=ya)
    torch.cuda.synchronize()
    del xa, ya
elif mode == "E":          # no autotune: allocate and free dummy blocks first
    p = vp.build_program(lay, pm, candidate=1)
    a = torch.empty(n, dtype=torch.uint8, device=dev)
    b = torch.empty(n, dtype=torch.uint8, device=dev)
    c = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    del a, b, c
if not pre:
    fl = bench.Flusher(torch, dev)
    x = torch.randint(0, 255, (n,), dtype=torch.uint8, device=dev)
    y = torch.empty_like(x)
st = torch.cuda.current_stream()
t = bench.time_device(torch, lambda: execute_device(p, x, out=y), 15, 3, fl, st)
t2 = bench.time_device(torch, lambda: execute_device(p, x, out=y), 15, 3, fl, st)
extra = ""
try:
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    extra = (f" mem {pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM)} MHz sm "
             f"{pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)} MHz temp "
             f"{pynvml.nvmlDeviceGetTemperature(h, pynvml.NVML_TEMPERATURE_GPU)} C pstate "
             f"{pynvml.nvmlDeviceGetPerformanceState(h)} reasons {pynvml.nvmlDeviceGetCurrentClocksEventReasons(h):#x}")
except Exception as e:
    extra = f" nvml: {e}"
print(mode + ("/pre" if pre else ""), p.metadata["src_run"], p.metadata["dst_run"], round(sorted(t)[7] * 1e3, 1), round(sorted(t2)[7] * 1e3, 1),
      extra)
