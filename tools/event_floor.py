"""How much of a flushed single-launch event time is fixed overhead?"""
import torch

dev = torch.device("cuda", 0)
st = torch.cuda.current_stream()
w = torch.empty(64 << 20, dtype=torch.float32, device=dev)
r = torch.zeros(64 << 20, dtype=torch.float32, device=dev)
one = torch.zeros(1, dtype=torch.int32, device=dev)
two = torch.zeros(1, dtype=torch.int32, device=dev)


def run(flush, work, n=30):
    ts = []
    for i in range(n + 5):
        flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        work()
        b.record(st)
        ts.append((a, b))
    torch.cuda.synchronize()
    v = sorted(a.elapsed_time(b) * 1e3 for a, b in ts[5:])
    return v[len(v) // 2]


flushes = {"none": lambda: None, "fill": lambda: w.fill_(1.0), "fill+sum": lambda: (w.fill_(1.0), r.sum()),
           "sum": lambda: r.sum(), "small": lambda: two.fill_(3)}
works = {"empty": lambda: None, "fill1": lambda: one.fill_(1), "fill1x2": lambda: (one.fill_(1), one.fill_(2))}
for fn, f in flushes.items():
    print(fn, {wn: round(run(f, wk), 2) for wn, wk in works.items()}, flush=True)

# CUDA-graph launch of the same tiny kernel: does the per-launch floor shrink?
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    one.fill_(1)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        one.fill_(1)
torch.cuda.synchronize()
for fn, f in [("fill", lambda: w.fill_(1.0)), ("none", lambda: None)]:
    print("graph", fn, {wn: round(run(f, wk), 2) for wn, wk in {"replay": lambda: g.replay()}.items()}, flush=True)
