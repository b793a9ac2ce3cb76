"""Sharded (multi-GPU) permutation logic on CPU: world_size 2 and 4 with the
gloo backend (127.0.0.1 rendezvous).  The exchange plan and the all-to-all
are the product's; the two local permutes are injected as numpy transposes
(the GPU kernels are covered by the -m gpu parity tests)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2506_03686_b200 import LayoutError
from paper_2506_03686_b200.sharded import plan_sharded, shard_bounds

CASES = [
    ((4, 6, 5), (2, 0, 1)),
    ((8, 3, 4), (1, 2, 0)),
    ((2,) * 10, (3, 9, 0, 7, 1, 5, 2, 8, 6, 4)),
    ((2,) * 12, (5, 11, 2, 7, 0, 9, 3, 1, 10, 4, 8, 6)),
    ((4, 4, 6), (0, 1, 2)),          # local only (I == O)
    ((4, 4, 6), (1, 0, 2)),          # pairwise exchange (same set, different order)
    ((12, 10, 4), (2, 1, 0)),
    ((16, 3, 2), (0, 2, 1)),
]


def _np_permute(x, axes):
    return torch.from_numpy(np.ascontiguousarray(np.transpose(x.numpy(), axes)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cases, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2506_03686_b200.sharded import permute_sharded

    errs = []
    for ci, (shape, axes) in enumerate(cases):
        try:
            rng = np.random.default_rng(ci)
            n = int(np.prod(shape))
            g = rng.integers(0, 2**62, size=n, dtype=np.int64)
            lo, hi = shard_bounds(n, world, rank)
            local = torch.from_numpy(g[lo:hi].copy())
            out = permute_sharded(local, shape, axes, local_permute=_np_permute)
            want = np.ascontiguousarray(np.transpose(g.reshape(shape), axes)).reshape(-1)[lo:hi]
            if not np.array_equal(out.numpy().reshape(-1), want):
                errs.append((shape, axes, "mismatch"))
        except LayoutError as e:
            errs.append((shape, axes, f"LayoutError {e}"))
    q.put((rank, errs))
    dist.barrier()
    dist.destroy_process_group()


def _run(world, cases):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    return res


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_gloo(world):
    cases = [c for c in CASES if _shardable(c, world)]
    assert len(cases) >= 5
    for rank, errs in _run(world, cases):
        assert not errs, (rank, errs)


def _shardable(case, G):
    try:
        plan_sharded(case[0], case[1], G)
        return True
    except LayoutError:
        return False


def test_plan_cfg5_structure():
    """Seed-0 cfg5 at G = 2/4/8 is a full all-to-all."""
    from paper_2506_03686_b200.workloads import CONFIGS

    wl = CONFIGS["cfg5"]
    for G in (2, 4, 8):
        sp = plan_sharded(wl.shape, wl.axes, G)
        sc = sp.send_counts(0)
        assert all(c == wl.numel // G // G for c in sc)
        assert sum(sp.recv_counts(3 % G)) == wl.numel // G
        assert len(sp.I) == len(sp.O) == {2: 1, 4: 2, 8: 3}[G]


def test_plan_local_and_pairwise():
    sp = plan_sharded((4, 4, 6), (0, 1, 2), 4)
    assert sp.send_counts(1) == [0, 24, 0, 0]                  # local only
    sp = plan_sharded((4, 4, 6), (1, 0, 2), 2)
    for r in range(2):
        assert sum(1 for c in sp.send_counts(r) if c) == 2      # halves exchanged
    with pytest.raises(LayoutError):
        plan_sharded((3, 5), (1, 0), 2)                        # not divisible
