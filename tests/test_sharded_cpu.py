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


def _worker(rank, world, port, cases, q, method="alltoall"):
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
            out = permute_sharded(local, shape, axes, local_permute=_np_permute, method=method)
            want = np.ascontiguousarray(np.transpose(g.reshape(shape), axes)).reshape(-1)[lo:hi]
            if not np.array_equal(out.numpy().reshape(-1), want):
                errs.append((shape, axes, "mismatch"))
        except LayoutError as e:
            errs.append((shape, axes, f"LayoutError {e}"))
    q.put((rank, errs))
    dist.barrier()
    dist.destroy_process_group()


def _run(world, cases, method="alltoall"):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q, method)) for r in range(world)]
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


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_gloo_pipelined(world):
    """The chunk-pipelined path (P1 chunk c+1 overlapping the all-to-all of
    chunk c, one P2 over the chunk-major receive buffer) over gloo."""
    from paper_2506_03686_b200.sharded import pipeline_chunks

    cases = [c for c in CASES + [((2,) * 14, (13, 4, 10, 11, 2, 0, 6, 12, 3, 7, 8, 1, 5, 9)),
                                 ((8, 12, 6, 4), (3, 1, 0, 2))] if _shardable(c, world)]
    assert sum(pipeline_chunks(plan_sharded(c[0], c[1], world)) > 1 for c in cases) >= 4
    for rank, errs in _run(world, cases, method="pipelined"):
        assert not errs, (rank, errs)


def test_pipeline_programs_emulated():
    """Chunked P1 programs, chunk-major receive layout and P2 program for
    virtual ranks (numpy local permutes), including every cfg5 shard count."""
    from paper_2506_03686_b200.sharded import emulate_sharded_pipelined, pipeline_chunks
    from paper_2506_03686_b200.workloads import CONFIGS

    cases = CASES + [((2,) * 14, (13, 4, 10, 11, 2, 0, 6, 12, 3, 7, 8, 1, 5, 9)), ((8, 12, 6, 4), (3, 1, 0, 2))]
    seen = 0
    for G in (2, 4, 8):
        for shape, axes in cases:
            if not _shardable((shape, axes), G):
                continue
            for chunks in (2, 4, 8):
                n = int(np.prod(shape))
                g = np.arange(n, dtype=np.int64)
                outs = emulate_sharded_pipelined(torch.from_numpy(g), shape, axes, G, local_permute=_np_permute,
                                                 chunks=chunks)
                want = np.ascontiguousarray(np.transpose(g.reshape(shape), axes)).reshape(-1)
                assert np.array_equal(torch.cat([o.reshape(-1) for o in outs]).numpy(), want), (G, shape, axes)
                seen += pipeline_chunks(plan_sharded(shape, axes, G), chunks) > 1
    assert seen >= 20
    w = CONFIGS["cfg5"]
    assert [pipeline_chunks(plan_sharded(w.shape, w.axes, G)) for G in (2, 4, 8)] == [4, 4, 2]


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
