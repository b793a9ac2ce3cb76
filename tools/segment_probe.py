"""Same-segment vs separate-segment src/dst for the cfg5 kernel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_03686_b200 as vp  # noqa: E402
from paper_2506_03686_b200.api import execute_device  # noqa: E402
from paper_2506_03686_b200.workloads import CONFIGS  # noqa: E402

mode = sys.argv[1]
wl = CONFIGS["cfg5"]
dev = torch.device("cuda", 0)
n = wl.numel * wl.elem_bytes
p = vp.build_program(vp.TensorLayout.from_shape(wl.shape, 8), vp.from_numpy_convention(wl.axes),
                     candidate=int(os.environ.get("CAND", "0")))
fl = bench.Flusher(torch, dev)
st = torch.cuda.current_stream()
if mode == "separate":
    x = torch.empty(n, dtype=torch.uint8, device=dev)
    y = torch.empty(n, dtype=torch.uint8, device=dev)
elif mode == "one":
    pool = torch.empty(2 * n, dtype=torch.uint8, device=dev)
    x, y = pool[:n], pool[n:]
elif mode in ("seed", "rand", "randn", "gen"):
    if mode == "seed":
        torch.cuda.manual_seed(0)
    elif mode == "rand":
        torch.rand(1024, device=dev)
    elif mode == "randn":
        torch.randn(1024, device=dev)
    else:
        torch.cuda.default_generators[0].initial_seed()
    x = torch.empty(n, dtype=torch.uint8, device=dev)
    y = torch.empty(n, dtype=torch.uint8, device=dev)
elif mode in ("smallalloc", "smallalloc_after"):
    if mode == "smallalloc":
        keep = torch.empty(1024, dtype=torch.uint8, device=dev)
    x = torch.empty(n, dtype=torch.uint8, device=dev)
    y = torch.empty(n, dtype=torch.uint8, device=dev)
    if mode == "smallalloc_after":
        keep = torch.empty(1024, dtype=torch.uint8, device=dev)
elif mode in ("tinyrand", "bigrand_other"):
    if mode == "tinyrand":
        torch.randint(0, 255, (1024,), dtype=torch.uint8, device=dev)
    else:
        z = torch.randint(0, 255, (n,), dtype=torch.uint8, device=dev)
        del z
    x = torch.empty(n, dtype=torch.uint8, device=dev)
    y = torch.empty(n, dtype=torch.uint8, device=dev)
elif mode.startswith("off"):
    # x, y as slices of one pool at a byte offset (VA / page alignment)
    off = int(mode[3:])
    pool = torch.empty(2 * n + 2 * off + (4 << 20), dtype=torch.uint8, device=dev)
    x, y = pool[off:off + n], pool[n + 2 * off:2 * n + 2 * off]
elif mode.startswith("pre"):
    # a big allocation first, released to the driver before x, y (physical placement)
    gb = int(mode[3:])
    z = torch.empty(gb << 30, dtype=torch.uint8, device=dev)
    del z
    torch.cuda.empty_cache()
    x = torch.empty(n, dtype=torch.uint8, device=dev)
    y = torch.empty(n, dtype=torch.uint8, device=dev)
elif mode.startswith("hold"):
    # a big allocation held while x, y are created
    gb = int(mode[4:])
    z = torch.empty(gb << 30, dtype=torch.uint8, device=dev)
    x = torch.empty(n, dtype=torch.uint8, device=dev)
    y = torch.empty(n, dtype=torch.uint8, device=dev)
elif mode in ("cumsum", "sort", "randint_after", "manual_seed_dev"):
    if mode == "cumsum":
        torch.ones(1024, device=dev).cumsum(0)
    elif mode == "sort":
        torch.ones(1024, device=dev).sort()
    elif mode == "manual_seed_dev":
        torch.cuda.manual_seed(0)
        torch.empty(16, device=dev).uniform_()
    x = torch.empty(n, dtype=torch.uint8, device=dev)
    y = torch.empty(n, dtype=torch.uint8, device=dev)
    if mode == "randint_after":
        torch.randint(0, 255, (1024,), dtype=torch.uint8, device=dev)
elif mode == "randint_late":
    x = torch.empty(n, dtype=torch.uint8, device=dev)
    y = torch.empty(n, dtype=torch.uint8, device=dev)
    execute_device(p, x, out=y)            # our specialised module loads first
    torch.cuda.synchronize()
    torch.randint(0, 255, (1024,), dtype=torch.uint8, device=dev)
elif mode == "randint":
    x = torch.randint(0, 255, (n,), dtype=torch.uint8, device=dev)
    y = torch.empty_like(x)
x.fill_(7)
t = bench.time_device(torch, lambda: execute_device(p, x, out=y), 15, 3, fl, st)
t2 = bench.time_device(torch, lambda: execute_device(p, x, out=y), 15, 3, fl, st)
print(mode, round(sorted(t)[7] * 1e3, 1), round(sorted(t2)[7] * 1e3, 1), hex(x.data_ptr()), hex(y.data_ptr()),
      torch.cuda.memory_reserved() >> 20, "MiB reserved", flush=True)
