"""Per-rank exchange kernel time on ONE GPU (all shards local): the fused
sharded kernels' own efficiency (push and pull), cfg5 at G = 1, 2, 4, 8.

Each rank's kernel reads 2 GiB / G and writes 2 GiB / G; on one GPU the
"remote" stores are local, so this bounds the kernel, not NVLink."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2506_03686_b200.api import launch_sharded, launch_sharded_pull  # noqa: E402
from paper_2506_03686_b200.sharded import _programs, shard_bounds  # noqa: E402
from paper_2506_03686_b200.workloads import CONFIGS  # noqa: E402

wl = CONFIGS["cfg5"]
dev = torch.device("cuda", 0)
fl = bench.Flusher(torch, dev)
st = torch.cuda.current_stream()
x = torch.randint(-2**62, 2**62, (wl.numel,), dtype=torch.int64, device=dev)
for mode in ("push", "pull"):
    for G in (1, 2, 4, 8):
        progs = _programs(wl.shape, wl.axes, 8, G, range(G), pull=mode == "pull")
        outs = [torch.empty(wl.numel // G, dtype=torch.int64, device=dev) for _ in range(G)]
        ptrs = [o.data_ptr() for o in outs]
        srcs = [x[shard_bounds(wl.numel, G, r)[0]:].data_ptr() for r in range(G)]
        sp = ctypes.c_void_p(st.cuda_stream)
        for r in (0, G - 1):
            if mode == "pull":
                fn = lambda: launch_sharded_pull(progs[r], srcs, ptrs[r], sp)  # noqa: E731
            else:
                fn = lambda: launch_sharded(progs[r], srcs[r], ptrs, sp)  # noqa: E731
            t = bench.time_device(torch, fn, 10, 3, fl, st)
            us = sorted(t)[len(t) // 2] * 1e3
            m = progs[r].metadata
            print(f"{mode} G={G} rank {r}: {us:7.1f} us  {wl.algorithmic_bytes / G / us / 1e3:6.0f} GB/s  "
                  f"tile {m['src_run']}x{m['dst_run']}", flush=True)
        del outs
