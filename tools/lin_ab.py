"""Paired A/B of two planner/kernel settings on random permutations (the
perf_sweep.py generator) plus named shapes: each shape is planned under
both settings (env knobs, plans rebuilt in-process), the launches are
interleaved, and the mean flushed time of each is reported with the ratio.
Shapes where both settings give the same plan text are skipped.

    python tools/lin_ab.py N seed "VPG_LIN=0" "VPG_LIN=1" [min_mib max_mib]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_03686_b200 as vp  # noqa: E402
from paper_2506_03686_b200.api import execute_device  # noqa: E402

N = int(sys.argv[1])
seed = int(sys.argv[2])
A = dict(kv.split("=") for kv in sys.argv[3].split()) if sys.argv[3] else {}
B = dict(kv.split("=") for kv in sys.argv[4].split()) if sys.argv[4] else {}
lo = int(sys.argv[5]) if len(sys.argv) > 5 else 16
hi = int(sys.argv[6]) if len(sys.argv) > 6 else 256
rng = np.random.default_rng(seed)
dev = torch.device("cuda", 0)
fl = bench.Flusher(torch, dev)
st = torch.cuda.current_stream()
pool = torch.empty(2 * (hi << 20), dtype=torch.uint8, device=dev)


def plan(env, lay, pm):
    keys = set(A) | set(B)
    for k in keys:
        os.environ.pop(k, None)
    os.environ.update(env)
    vp.program_cache_clear()
    p = vp.build_program(lay, pm)
    for k in keys:
        os.environ.pop(k, None)
    return p


def shapes():
    yield (17, 9, 13, 15, 11, 27), (5, 2, 0, 4, 1, 3), 4
    yield (7, 9, 13, 5, 11, 13, 9), (6, 2, 0, 4, 1, 3, 5), 4
    yield (267, 701, 717), (2, 1, 0), 4
    yield (131, 93, 77, 31), (3, 1, 2, 0), 8
    yield (4096, 4096), (1, 0), 4
    yield (32, 64, 56, 56), (0, 2, 3, 1), 4
    yield (8, 2, 5, 158, 37, 143), (2, 1, 0, 5, 4, 3), 4
    for _ in range(N):
        E = int(rng.choice([4, 8]))
        target = int(rng.integers(lo, hi + 1)) << 20
        r = int(rng.integers(2, 8))
        n = target // E
        dims, rem = [], n
        for k in range(r - 1):
            h = max(2, int(round(rem ** (1.0 / (r - k)) * rng.uniform(0.5, 2.0))))
            d = int(rng.integers(2, h + 1))
            if rng.random() < 0.5:
                d = d | 1
            dims.append(d)
            rem = max(1, rem // d)
        dims.append(max(2, rem))
        yield tuple(dims), tuple(int(a) for a in rng.permutation(r)), E


rat, srat = [], []
for shape, axes, E in shapes():
    nbytes = int(np.prod(shape)) * E
    if nbytes > (hi << 20):
        continue
    lay, pm = vp.TensorLayout.from_shape(shape, E), vp.from_numpy_convention(axes)
    pa, pb = plan(A, lay, pm), plan(B, lay, pm)
    # (knobs that only change the specialised kernel's source keep the plan text)
    if (pa.text == pb.text and not (set(A) | set(B)) & {"VPG_FLAT", "VPG_HINTS"}) or pa.kernel != "tile":
        continue
    if pa.text == pb.text and not any(ln.startswith("vector elems") and ln.endswith("W 1") for ln in pa.text.splitlines()):
        continue    # (flat walk: scalar W phases only)
    x, y = pool[:nbytes], pool[hi << 20:(hi << 20) + nbytes]
    ta, tb = [], []
    for _ in range(3):
        ta += bench.time_device(torch, lambda: execute_device(pa, x, out=y), 5, 1, fl, st)
        tb += bench.time_device(torch, lambda: execute_device(pb, x, out=y), 5, 1, fl, st)
    ma, mb = np.mean(ta) * 1e3, np.mean(tb) * 1e3
    rat.append(ma / mb)
    lin_b = "W lin" in pb.text
    extra = ""
    if os.environ.get("AB_STEADY"):
        # back-to-back over rotating buffers larger than L2 (bench.time_steady)
        nb = bench.steady_buffers(fl.l2, nbytes)
        xs = [torch.empty(nbytes, dtype=torch.uint8, device=dev) for _ in range(nb)]
        ys = [torch.empty(nbytes, dtype=torch.uint8, device=dev) for _ in range(nb)]
        reps = max(3, min(30, int(4e9 // (nb * 2 * nbytes))))
        sa = min(bench.time_steady(torch, lambda i: execute_device(pa, xs[i], out=ys[i]), nb, reps, st) for _ in range(3))
        sb = min(bench.time_steady(torch, lambda i: execute_device(pb, xs[i], out=ys[i]), nb, reps, st) for _ in range(3))
        srat.append(sa / sb)
        extra = f" | steady A {sa * 1e3:8.2f} B {sb * 1e3:8.2f} A/B {sa / sb:.3f}"
        del xs, ys
    print(f"{shape} {axes} E={E} runs {pa.metadata['src_run']}x{pa.metadata['dst_run']} | "
          f"{pb.metadata['src_run']}x{pb.metadata['dst_run']} lin_b={int(lin_b)}: A {ma:8.2f} us  B {mb:8.2f} us  "
          f"A/B {ma / mb:.3f}  ({2 * nbytes / mb / 1e3:6.0f} GB/s B){extra}", flush=True)
r = np.array(rat)
if r.size:
    print(f"\n{r.size} shapes: A/B time ratio median {np.median(r):.3f} p10 {np.percentile(r, 10):.3f} "
          f"p90 {np.percentile(r, 90):.3f} min {r.min():.3f} max {r.max():.3f}  (>1: B faster)")
if srat:
    r = np.array(srat)
    print(f"steady: A/B time ratio median {np.median(r):.3f} p10 {np.percentile(r, 10):.3f} "
          f"p90 {np.percentile(r, 90):.3f} min {r.min():.3f} max {r.max():.3f}")
