"""Launch each BASELINE config's kernel twice inside an NVTX range
"capture", with the plans bench.py uses (the cost model's), for ncu:

  ncu --set full --clock-control none --import-source on --nvtx \
      --nvtx-include "capture/" -o gpurun_out/full_rN python tools/profile_configs.py

Order: cfg5, cfg4, cfg3, cfg1, cfg2, then the cfg5 push exchange kernel
of rank 0 of 2 (label cfg5/2) and the cfg5 pull exchange kernel of rank 0
of 8 (label cfg5/8p; all shards local); labels for tools/ncu_summary.py."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_03686_b200 as vp  # noqa: E402
from paper_2506_03686_b200.api import execute_device  # noqa: E402
from paper_2506_03686_b200.workloads import CONFIGS  # noqa: E402

ORDER = ["cfg5", "cfg4", "cfg3", "cfg1", "cfg2"]
dev = torch.device("cuda", 0)
runs = []
for k in ORDER:
    wl = CONFIGS[k]
    prog = vp.build_program(vp.TensorLayout.from_shape(wl.shape, wl.elem_bytes), vp.from_numpy_convention(wl.axes))
    n = wl.numel * wl.elem_bytes
    x = torch.randint(0, 255, (n,), dtype=torch.uint8, device=dev)
    y = torch.empty_like(x)
    execute_device(prog, x, out=y)          # compile/load outside the capture
    runs.append((k, prog, x, y))
    print(k, prog.kernel, prog.metadata["src_run"], prog.metadata["dst_run"], flush=True)
# the fused sharded exchange kernel of rank 0 of 2 (cfg5), both output
# shards local (tools/exchange_probe.py): label "cfg5/2"
import ctypes  # noqa: E402

from paper_2506_03686_b200.api import launch_sharded, launch_sharded_pull  # noqa: E402
from paper_2506_03686_b200.sharded import _programs, shard_bounds  # noqa: E402

wl5 = CONFIGS["cfg5"]
xprog = _programs(wl5.shape, wl5.axes, 8, 2, [0])[0]
x5 = runs[0][2]
outs = [torch.empty(wl5.numel * 8 // 2, dtype=torch.uint8, device=dev) for _ in range(2)]
sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
launch_sharded(xprog, x5.data_ptr(), [o.data_ptr() for o in outs], sp)
pprog = _programs(wl5.shape, wl5.axes, 8, 8, [0], pull=True)[0]
psrcs = [x5.data_ptr() + shard_bounds(wl5.numel, 8, r)[0] * 8 for r in range(8)]
pout = torch.empty(wl5.numel * 8 // 8, dtype=torch.uint8, device=dev)
launch_sharded_pull(pprog, psrcs, pout.data_ptr(), sp)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("capture")
for k, prog, x, y in runs:
    for _ in range(2):
        execute_device(prog, x, out=y)
for _ in range(2):
    launch_sharded(xprog, x5.data_ptr(), [o.data_ptr() for o in outs], sp)
for _ in range(2):
    launch_sharded_pull(pprog, psrcs, pout.data_ptr(), sp)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
