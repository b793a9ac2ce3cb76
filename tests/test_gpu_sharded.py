"""Sharded permutation with the real GPU kernels in separate processes.

Two (or four) ranks share the one GPU of the test box; their P1/P2
permutes run as independent GPU kernels and the exchange runs over the
gloo process group (device data staged through host memory).  No kernel
waits on another rank.  The NCCL transport used on multi-GPU boxes is the
same all_to_all_single call on device buffers."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [
    ((2,) * 20, (19, 4, 10, 11, 2, 17, 6, 16, 3, 0, 8, 1, 18, 12, 14, 13, 7, 5, 15, 9)),
    ((8, 6, 10, 4), (2, 0, 3, 1)),
    ((16, 12, 17, 9), (3, 1, 0, 2)),
    ((4, 64, 128), (2, 1, 0)),
]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2506_03686_b200.sharded import permute_sharded, plan_sharded, shard_bounds

    errs = []
    for ci, (shape, axes) in enumerate(CASES):
        try:
            plan_sharded(shape, axes, world)
        except Exception:
            continue
        n = int(np.prod(shape))
        g = np.random.default_rng(ci).integers(-2**62, 2**62, size=n, dtype=np.int64)
        lo, hi = shard_bounds(n, world, rank)
        local = torch.from_numpy(g[lo:hi].copy()).cuda()
        out = permute_sharded(local, shape, axes)           # GPU kernels for P1 and P2
        torch.cuda.synchronize()
        want = np.ascontiguousarray(np.transpose(g.reshape(shape), axes)).reshape(-1)[lo:hi]
        if not np.array_equal(out.cpu().numpy().reshape(-1), want):
            errs.append((shape, axes))
    q.put((rank, errs))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_ranks_with_gpu_kernels(cuda, world):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
    for rank, errs in res:
        assert not errs, (rank, errs)
