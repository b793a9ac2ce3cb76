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


def _fused_worker(rank, world, port, q, mode="push"):
    """Fused exchange (ShardExchange): CUDA IPC peer table between processes
    sharing the GPU; each rank's kernel stores into the others' output
    buffers (push) or reads the others' input buffers (pull)."""
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2506_03686_b200.sharded import ShardExchange, permute_sharded, shard_bounds

    errs, ran, live = [], 0, []
    for ci, (shape, axes) in enumerate(FUSED_CASES):
        try:
            ex = ShardExchange(shape, axes, torch.int64, mode=mode)
        except Exception as e:          # shapes that do not shard over `world`
            if "unsupported" not in str(e):
                errs.append((shape, axes, repr(e)))
            continue
        n = int(np.prod(shape))
        g = np.random.default_rng(ci).integers(-2**62, 2**62, size=n, dtype=np.int64)
        lo, hi = shard_bounds(n, world, rank)
        want = np.ascontiguousarray(np.transpose(g.reshape(shape), axes)).reshape(-1)[lo:hi]
        for step in range(2):           # the second call reuses the mapped buffers
            local = torch.from_numpy(g[lo:hi].copy()).cuda()
            out = ex(local)
            torch.cuda.synchronize()
            if not np.array_equal(out.cpu().numpy().reshape(-1), want):
                errs.append((shape, axes, step))
        # results of consecutive calls do not alias (push: alternating
        # registered outputs; pull: a fresh output per call)
        o1 = ex(local)
        o2 = ex(local)
        torch.cuda.synchronize()
        if o1.data_ptr() == o2.data_ptr() or not (np.array_equal(o1.cpu().numpy().reshape(-1), want)
                                                   and np.array_equal(o2.cpu().numpy().reshape(-1), want)):
            errs.append((shape, axes, "consecutive results"))
        if mode == "pull":              # the registered input buffer: no staging copy
            buf = ex.input_buffer()
            buf.copy_(local)
            o3 = ex(buf)
            torch.cuda.synchronize()
            if not np.array_equal(o3.cpu().numpy().reshape(-1), want):
                errs.append((shape, axes, "registered input"))
        # permute_sharded(method="fused") builds its own cached exchange (a second mapping of the peers)
        out = permute_sharded(torch.from_numpy(g[lo:hi].copy()).cuda(), shape, axes, method="fused")
        torch.cuda.synchronize()
        if not np.array_equal(out.cpu().numpy().reshape(-1), want):
            errs.append((shape, axes, "permute_sharded"))
        live.append((ex, local, want))  # exchanges stay mapped together (shared allocator segments)
        ran += 1
    for ex, local, want in live:        # every exchange still works with all mappings open
        out = ex(local)
        torch.cuda.synchronize()
        if not np.array_equal(out.cpu().numpy().reshape(-1), want):
            errs.append(("live", ex.splan.shape))
    for ex, _, _ in live:
        ex.close()
    q.put((rank, errs, ran))
    dist.barrier()
    dist.destroy_process_group()


FUSED_CASES = [
    ((2,) * 20, (19, 4, 10, 11, 2, 17, 6, 16, 3, 0, 8, 1, 18, 12, 14, 13, 7, 5, 15, 9)),
    ((8, 6, 16, 4), (2, 0, 3, 1)),
    ((8, 40, 32), (0, 2, 1)),
    ((2, 16, 6, 16, 4, 8), (3, 2, 0, 1, 4, 5)),
    ((8, 8, 24, 10), (1, 3, 0, 2)),
]


@pytest.mark.parametrize("mode", ["push", "pull"])
@pytest.mark.parametrize("world", [2, 4])
def test_fused_exchange_processes(cuda, world, mode):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fused_worker, args=(r, world, port, q, mode)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
    for rank, errs, ran in res:
        assert not errs, (rank, errs)
        assert ran >= 3, (rank, ran)


@pytest.mark.parametrize("mode", ["push", "pull"])
@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_fused_exchange_emulated(cuda, G, mode):
    """All G exchange kernels on one device (independent launches into G
    local output shards): bit-exact against numpy."""
    import torch

    import paper_2506_03686_b200 as vp
    from paper_2506_03686_b200.sharded import emulate_fused

    ran = 0
    for ci, (shape, axes) in enumerate(FUSED_CASES + CASES):
        n = int(np.prod(shape))
        g = np.random.default_rng(100 + ci).integers(-2**62, 2**62, size=n, dtype=np.int64)
        try:
            outs = emulate_fused(torch.from_numpy(g).cuda(), shape, axes, G, mode=mode)
        except vp.LayoutError:
            continue
        torch.cuda.synchronize()
        got = torch.cat(outs).cpu().numpy()
        assert np.array_equal(got, np.ascontiguousarray(np.transpose(g.reshape(shape), axes)).reshape(-1)), (shape, axes)
        ran += 1
    assert ran >= 3


@pytest.mark.parametrize("mode", ["push", "pull"])
@pytest.mark.parametrize("G", [2, 4, 8])
def test_fused_exchange_cfg5(cuda, G, mode):
    """BASELINE cfg5 (2 GiB) through the G exchange kernels on one device,
    compared with the single-GPU permutation (itself pinned to the oracle in
    test_gpu_configs) and the closed-form bijection on sampled positions."""
    import torch

    from paper_2506_03686_b200 import permute
    from paper_2506_03686_b200.sharded import emulate_fused
    from paper_2506_03686_b200.workloads import CONFIGS

    w = CONFIGS["cfg5"]
    x = torch.randint(-2**62, 2**62, (w.numel,), dtype=torch.int64, device="cuda",
                      generator=torch.Generator(device="cuda").manual_seed(G))
    outs = emulate_fused(x, w.shape, w.axes, G, mode=mode)
    whole = permute(x.view(w.shape), w.axes).reshape(-1)
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(outs), whole)
    # sampled closed-form check: out[i] = in[f(i)]
    idx = torch.randint(0, w.numel, (1 << 16,), device="cuda")
    src = torch.zeros_like(idx)
    rem = idx.clone()
    in_strides = [1 << (27 - k) for k in range(28)]
    for a in reversed(w.axes):
        src += (rem % 2) * in_strides[a]
        rem //= 2
    assert torch.equal(torch.cat(outs)[idx], x[src])


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


@pytest.mark.parametrize("dtype_name,jit", [("uint8", False), ("int16", False), ("int32", True), ("int32", False),
                                            ("float64", True), ("complex128", False)])
@pytest.mark.parametrize("mode", ["push", "pull"])
def test_fused_exchange_word_sizes(cuda, dtype_name, jit, mode):
    """1/2/4/8/16-byte words through both the specialised and the
    ahead-of-time exchange kernels (emulated ranks on one device)."""
    import torch

    import paper_2506_03686_b200 as vp
    from paper_2506_03686_b200.sharded import emulate_fused

    tdt = getattr(torch, dtype_name)
    ran = 0
    for ci, (shape, axes) in enumerate(FUSED_CASES):
        n = int(np.prod(shape))
        g = torch.Generator().manual_seed(ci)
        x = (torch.randint(-100, 100, (n,), generator=g).to(tdt) if not tdt.is_complex
             else torch.randn(n, dtype=tdt, generator=g))
        for G in (2, 4):
            try:
                outs = emulate_fused(x.cuda(), shape, axes, G, jit=jit, mode=mode)
            except vp.LayoutError:
                continue
            got = torch.cat(outs).cpu()
            assert torch.equal(got, x.reshape(shape).permute(axes).reshape(-1)), (shape, axes, G)
            ran += 1
    assert ran >= 4


@pytest.mark.parametrize("method", ["push", "pull", "alltoall", "pipelined"])
def test_bench_two_ranks_code_path(cuda, method):
    """bench.py's N>1 path (torchrun, two ranks) end to end with the gloo
    backend on one GPU: the same code the 8-GPU NCCL run takes, checked for
    per-rank sampled parity (timings of this run are not multi-GPU results)."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
           "--dist-backend", "gloo", "--shard-method", method, "--config", "cfg1", "--steps", "2", "--warmup", "3"]
    res = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    line = json.loads([ln for ln in res.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["parity_sampled"] is True
    assert line["shard_method"] == (method if method in ("alltoall", "pipelined") else f"fused ({method})")
    assert line["n_gpus"] == 2
    assert "gloo" in line["dist_backend"]


def test_bench_two_ranks_fused_fallback(cuda):
    """A fused exchange that fails its pre-flight check on any rank (forced
    here) makes every rank fall back to the NCCL-style all-to-all path, and
    the JSON line records why."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
           "--dist-backend", "gloo", "--config", "cfg1", "--steps", "2", "--warmup", "3"]
    env = dict(os.environ, VPG_BENCH_FORCE_FUSED_FAIL="1")
    res = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=600, env=env)
    assert res.returncode == 0, res.stderr[-2000:]
    line = json.loads([ln for ln in res.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["parity_sampled"] is True and line["e2e"]["parity"] is True
    assert line["shard_method"] in ("alltoall", "pipelined")
    assert "forced" in line["fused_exchange_fallback"]


@pytest.mark.parametrize("mode", ["push", "pull"])
def test_fused_exchange_random_campaign(cuda, mode):
    """Random shapes (factors of 2, 3, 4, 6, 8, 12, 16), ranks 2-7, words of
    4 and 8 bytes, G in {2, 4, 8}: every exchange plan that exists is
    bit-exact against numpy (emulated ranks on one device)."""
    import torch

    import paper_2506_03686_b200 as vp
    from paper_2506_03686_b200.sharded import emulate_fused

    rng = np.random.default_rng(2024)
    ran = 0
    for it in range(300):
        r = int(rng.integers(2, 8))
        shape = tuple(int(x) for x in rng.choice([2, 3, 4, 6, 8, 12, 16], size=r))
        if int(np.prod(shape)) > (1 << 20):
            continue
        axes = tuple(int(a) for a in rng.permutation(r))
        G = int(rng.choice([2, 4, 8]))
        dt = torch.int32 if it % 2 else torch.int64
        n = int(np.prod(shape))
        x = torch.randint(-2**31, 2**31 - 1, (n,), dtype=dt, device="cuda")
        try:
            outs = emulate_fused(x, shape, axes, G, mode=mode)
        except vp.LayoutError:
            continue
        got = torch.cat(outs)
        assert torch.equal(got, x.view(shape).permute(axes).reshape(-1)), (shape, axes, G)
        ran += 1
    assert ran >= 100, ran


@pytest.mark.parametrize("offset_words", [0, 1])
def test_pull_exchange_separate_buffers(cuda, offset_words):
    """Pull exchange with every input shard in its own allocation (as with
    peer-mapped buffers), including shard buffers off 16-byte alignment
    (offset_words = 1: the plan's scalar-read variant must take over)."""
    import torch

    import paper_2506_03686_b200 as vp
    from paper_2506_03686_b200.sharded import emulate_fused, shard_bounds

    ran = 0
    for shape, axes, G in [((2,) * 20, CASES[0][1], 4), ((2,) * 20, CASES[0][1], 8), ((8, 6, 16, 4), (2, 0, 3, 1), 2),
                           ((16, 12, 16, 8), (3, 1, 0, 2), 4), ((8, 40, 32), (0, 2, 1), 2)]:
        n = int(np.prod(shape))
        x = torch.randint(-2**31, 2**31 - 1, (n,), dtype=torch.int32, device="cuda")
        shards = []
        for r in range(G):
            lo, hi = shard_bounds(n, G, r)
            buf = torch.empty(hi - lo + 4, dtype=torch.int32, device="cuda")
            v = buf[offset_words:offset_words + hi - lo]
            v.copy_(x[lo:hi])
            shards.append(v)
        try:
            outs = emulate_fused(x, shape, axes, G, mode="pull", in_shards=shards)
        except vp.LayoutError:          # no pull plan for this shape
            continue
        assert torch.equal(torch.cat(outs), x.view(shape).permute(axes).reshape(-1)), (shape, axes, G)
        ran += 1
    assert ran >= 3


def test_pull_exchange_nonpow2_shards_beyond_32bit_offsets(cuda):
    """Pull exchange with G = 3 (shard size not a power of two) on more than
    2^32 one-byte elements: the source shard of every chunk is found with a
    64-bit divide (tile_body.cuh pull_ptr); a 32-bit one would read the wrong
    shard past offset 2^32."""
    import torch

    import paper_2506_03686_b200 as vp
    from paper_2506_03686_b200.sharded import emulate_fused, shard_bounds

    shape, axes, G = (3, 1 << 21, 768), (2, 1, 0), 3
    n = 3 * (1 << 21) * 768
    assert n > 1 << 32
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda", generator=g)
    shards = [x[slice(*shard_bounds(n, G, r))].clone() for r in range(G)]
    try:
        outs = emulate_fused(x, shape, axes, G, mode="pull", in_shards=shards)
    except vp.LayoutError as e:
        pytest.skip(f"no pull plan: {e}")
    del shards
    torch.cuda.synchronize()
    want = x.view(shape).permute(axes).contiguous().reshape(-1)
    got = torch.cat(outs)
    assert torch.equal(got, want)


@pytest.mark.parametrize("G", [2, 4, 8])
def test_pipelined_alltoall_cfg5_emulated(cuda, G):
    """The chunk-pipelined all-to-all path's GPU programs on cfg5 (2 GiB):
    chunked P1 kernels, chunk-major receive buffers and the P2 kernel for G
    virtual ranks on one device, against the single-GPU permutation."""
    import torch

    from paper_2506_03686_b200 import permute
    from paper_2506_03686_b200.sharded import emulate_sharded_pipelined, pipeline_chunks, plan_sharded
    from paper_2506_03686_b200.workloads import CONFIGS

    w = CONFIGS["cfg5"]
    assert pipeline_chunks(plan_sharded(w.shape, w.axes, G)) > 1
    x = torch.randint(-2**62, 2**62, (w.numel,), dtype=torch.int64, device="cuda",
                      generator=torch.Generator(device="cuda").manual_seed(10 + G))
    outs = emulate_sharded_pipelined(x, w.shape, w.axes, G)
    whole = permute(x.view(w.shape), w.axes).reshape(-1)
    torch.cuda.synchronize()
    assert torch.equal(torch.cat([o.reshape(-1) for o in outs]), whole)


@pytest.mark.parametrize("mode", ["push", "pull"])
@pytest.mark.parametrize("G", [2, 4, 8])
def test_fused_exchange_device_barrier_emulated(cuda, G, mode):
    """The device-side exchange barrier (flag blocks, epochs; no collective
    around the launch): all G ranks' kernels in ONE cooperative launch on
    this GPU, exactly the kernel code a multi-GPU job runs per rank through
    vpg_permute_sharded_sync.  Bit-exact against the single-GPU permutation
    on cfg5 and on small shapes with ragged tiles."""
    import torch

    from paper_2506_03686_b200 import LayoutError, permute
    from paper_2506_03686_b200.sharded import emulate_fused
    from paper_2506_03686_b200.workloads import CONFIGS

    w = CONFIGS["cfg5"]
    cases = [(w.shape, w.axes)] + list(FUSED_CASES)
    ran = 0
    for ci, (shape, axes) in enumerate(cases):
        n = 1
        for d in shape:
            n *= d
        x = torch.randint(-2**62, 2**62, (n,), dtype=torch.int64, device="cuda",
                          generator=torch.Generator(device="cuda").manual_seed(100 + ci))
        try:
            outs = emulate_fused(x, shape, axes, G, mode=mode, device_barrier=True)
        except LayoutError:
            continue                      # no exchange plan for this shape / G
        whole = permute(x.view(shape), axes).reshape(-1)
        torch.cuda.synchronize()
        assert torch.equal(torch.cat(outs), whole), (shape, axes, G, mode)
        ran += 1
    assert ran >= 2
