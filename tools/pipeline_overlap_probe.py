"""Overlap evidence for the chunk-pipelined all-to-all path on ONE GPU.

G virtual ranks (cfg5, 2 GiB): per chunk c, the P1 kernels of every rank run
on the compute stream; the chunk's exchange is emulated by device-to-device
copies on a second stream (the copy engines stand in for NCCL over NVLink);
P1 of chunk c+1 overlaps the copies of chunk c.  One P2 per rank at the end.
Prints the serial and pipelined step times and the per-chunk timeline (CUDA
events), and checks the result against the single-GPU permutation.  No
kernel waits on another (stream events only)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2506_03686_b200 import permute  # noqa: E402
from paper_2506_03686_b200.sharded import (_pipelined_programs, pipeline_chunks, pipeline_spec,  # noqa: E402
                                           plan_sharded, shard_bounds)
from paper_2506_03686_b200.workloads import CONFIGS  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 4
w = CONFIGS["cfg5"]
dev = torch.device("cuda", 0)
sp = plan_sharded(w.shape, w.axes, G)
spec = pipeline_spec(sp)
C = pipeline_chunks(sp)
(s1c, a1), (s2c, a2c) = _pipelined_programs(sp, spec)
n = w.numel
x = torch.randint(-2**62, 2**62, (n,), dtype=torch.int64, device=dev, generator=torch.Generator(device=dev).manual_seed(1))
shard = n // G
packed = [[torch.empty(shard // C, dtype=torch.int64, device=dev) for _ in range(C)] for _ in range(G)]
recv = [torch.empty(shard, dtype=torch.int64, device=dev) for _ in range(G)]
outs = [torch.empty(shard, dtype=torch.int64, device=dev) for _ in range(G)]
send = [[k // C for k in sp.send_counts(r)] for r in range(G)]
comp, comm = torch.cuda.current_stream(dev), torch.cuda.Stream(dev)


def ev(st):
    e = torch.cuda.Event(enable_timing=True)
    e.record(st)
    return e


def step(pipelined, marks):
    chunk_done = []
    for c in range(C):
        t0 = ev(comp)
        for r in range(G):
            lo, _ = shard_bounds(n, G, r)
            xin = x[lo:lo + shard].view(C, -1)[c]
            permute(xin.view(s1c), a1, out=packed[r][c].view([s1c[i] for i in a1]))
        t1 = ev(comp)
        chunk_done.append(t1)
        marks.append(("P1", c, t0, t1))
    if pipelined:
        # every P1 chunk is queued first (the host issues the emulated
        # exchange copies one by one; NCCL's all-to-all is one call): the
        # copies of chunk c start when its P1 finishes, under P1 of c+1
        for c in range(C):
            comm.wait_event(chunk_done[c])
            with torch.cuda.stream(comm):
                t2 = ev(comm)
                copy_chunk(c)
                marks.append(("xchg", c, t2, ev(comm)))
    else:
        comm.wait_event(chunk_done[-1])
        with torch.cuda.stream(comm):
            for c in range(C):
                t2 = ev(comm)
                copy_chunk(c)
                marks.append(("xchg", c, t2, ev(comm)))
    comp.wait_stream(comm)
    t3 = ev(comp)
    for s in range(G):
        permute(recv[s].view(s2c), a2c, out=outs[s].view([s2c[i] for i in a2c]))
    marks.append(("P2", -1, t3, ev(comp)))


def copy_chunk(c):
    # recv[s] is chunk-major: [c][source r][block]
    for s in range(G):
        base = c * (shard // C)
        off_r = 0
        for r in range(G):
            k = send[r][s]
            if k:
                src_off = sum(send[r][:s])
                recv[s][base + off_r:base + off_r + k].copy_(packed[r][c][src_off:src_off + k], non_blocking=True)
                off_r += k


res = {}
for mode in ("serial", "pipelined", "serial", "pipelined"):
    marks = []
    torch.cuda.synchronize()
    a = ev(comp)
    step(mode == "pipelined", marks)
    b = ev(comp)
    torch.cuda.synchronize()
    tl = [(k, c, round(a.elapsed_time(s), 3), round(a.elapsed_time(e), 3)) for k, c, s, e in marks]
    res[mode] = {"step_ms": round(a.elapsed_time(b), 3), "timeline_ms": tl}
whole = permute(x.view(w.shape), w.axes).reshape(-1)
torch.cuda.synchronize()
ok = bool(torch.equal(torch.cat(outs), whole))
print(json.dumps({"G": G, "chunks": C, "spec": spec, "parity": ok, **res}))
