"""Cross-PROCESS check of the device-side exchange barrier: two ranks (gloo
for the IPC handle exchange only) share this one GPU; each ShardExchange
call launches one kernel per rank that signals/waits on the other rank's
flag block through CUDA IPC.  Without MPS the two contexts time-slice, so
the waits complete at context switches (slow, but every wait is bounded by
~4 s -- the device cannot hang).  Prints per-call wall time and parity.
On a multi-GPU node each rank has its own GPU and no time-slicing occurs."""
import os
import socket
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def worker(rank, world, port, mode, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2506_03686_b200.sharded import ShardExchange, shard_bounds

    shape, axes = (8, 6, 16, 4), (2, 0, 3, 1)
    n = int(np.prod(shape))
    g = np.random.default_rng(0).integers(-2**62, 2**62, size=n, dtype=np.int64)
    lo, hi = shard_bounds(n, world, rank)
    want = np.ascontiguousarray(np.transpose(g.reshape(shape), axes)).reshape(-1)[lo:hi]
    ex = ShardExchange(shape, axes, torch.int64, mode=mode, device_barrier=True)
    local = torch.from_numpy(g[lo:hi].copy()).cuda()
    res = []
    for step in range(3):
        dist.barrier()
        t0 = time.perf_counter()
        out = ex(local)
        torch.cuda.synchronize()
        res.append((round(time.perf_counter() - t0, 4), bool(np.array_equal(out.cpu().numpy().reshape(-1), want))))
    q.put((rank, mode, res))
    dist.barrier()
    ex.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    for mode in ("push", "pull"):
        q = ctx.Queue()
        port = _port()
        ps = [ctx.Process(target=worker, args=(r, 2, port, mode, q)) for r in range(2)]
        for p in ps:
            p.start()
        for _ in ps:
            print(q.get(timeout=300), flush=True)
        for p in ps:
            p.join(timeout=60)
