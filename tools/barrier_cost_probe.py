"""Cost of the device-side exchange barrier: cfg5 (2 GiB) exchange steps of
G virtual ranks in one cooperative launch, with the barrier (flag blocks,
epochs) and without it (VPG_EMU_NO_BARRIER=1 in a second process), plus
the G independent launches of the same plans for reference.  Wall time of
the (synchronous) emulation call, median of 7."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2506_03686_b200.sharded import emulate_fused  # noqa: E402
from paper_2506_03686_b200.workloads import CONFIGS  # noqa: E402

w = CONFIGS["cfg5"]
x = torch.randint(-2**62, 2**62, (w.numel,), dtype=torch.int64, device="cuda")
for G, mode in ((2, "push"), (4, "push"), (8, "push"), (2, "pull"), (4, "pull"), (8, "pull")):
    res = {}
    for coop in (True, False):
        ts = []
        for i in range(9):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            outs = emulate_fused(x, w.shape, w.axes, G, mode=mode, device_barrier=coop)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
            del outs
        res["cooperative" if coop else "independent"] = round(sorted(ts[2:])[3] * 1e3, 3)
    print(f"G={G} {mode} barrier={'off' if os.environ.get('VPG_EMU_NO_BARRIER') else 'on'} ms {res}", flush=True)
