"""Decompose the ~6 us event floor of a flushed single launch on B200:
which part is the event pair, which the first kernel after an event, and
does a preceding tiny kernel (or PDL) change it?"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

dev = torch.device("cuda", 0)
st = torch.cuda.current_stream()
fl = bench.Flusher(torch, dev)
one = torch.zeros(1, dtype=torch.int32, device=dev)
two = torch.zeros(1, dtype=torch.int32, device=dev)
big = torch.empty(64 << 20, dtype=torch.uint8, device=dev)
bigo = torch.empty_like(big)


def t(pre, work, n=40):
    for _ in range(3):
        pre()
        work()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    torch.cuda._sleep(40_000_000)
    for a, b in evs:
        pre()
        a.record(st)
        work()
        b.record(st)
    torch.cuda.synchronize()
    v = sorted(a.elapsed_time(b) * 1e3 for a, b in evs)
    return round(v[len(v) // 2], 2)


nothing = lambda: None  # noqa: E731
fill1 = lambda: one.fill_(1)  # noqa: E731
fill2 = lambda: (one.fill_(1), two.fill_(2))  # noqa: E731
fill3 = lambda: (one.fill_(1), two.fill_(2), one.fill_(3))  # noqa: E731
copy64 = lambda: bigo.copy_(big)  # noqa: E731
copy64x2 = lambda: (bigo.copy_(big), bigo.copy_(big))  # noqa: E731
for pn, pre in [("noflush", nothing), ("flush", fl), ("flush+fill", lambda: (fl(), two.fill_(5)))]:
    print(pn, {wn: t(pre, w) for wn, w in [("empty", nothing), ("fill1", fill1), ("fill2", fill2),
                                           ("fill3", fill3), ("copy64M", copy64), ("copy64Mx2", copy64x2)]},
          flush=True)
