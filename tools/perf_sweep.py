"""Performance over random large permutations (64-512 MiB, ranks 2-8,
4/8-byte words): flushed single launches vs same-size copy_; prints the
distribution and the worst cases (to find planner/kernel cliffs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_03686_b200 as vp  # noqa: E402
from paper_2506_03686_b200.api import execute_device  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 60
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
rng = np.random.default_rng(seed)
dev = torch.device("cuda", 0)
fl = bench.Flusher(torch, dev)
st = torch.cuda.current_stream()
pool = torch.empty(2 * (512 << 20), dtype=torch.uint8, device=dev)
rows = []
for i in range(N):
    E = int(rng.choice([int(w) for w in os.environ.get("SWEEP_WORDS", "4,8").split(",")]))
    target = int(rng.choice([64, 128, 256, 512])) << 20
    r = int(rng.integers(2, 9))
    # random factorisation of target/E elements into r dims (mix of odd and even extents)
    n = target // E
    dims = []
    rem = n
    for k in range(r - 1):
        hi = max(2, int(round(rem ** (1.0 / (r - k)) * rng.uniform(0.5, 2.0))))
        d = int(rng.integers(2, hi + 1))
        if rng.random() < 0.3:
            d = d | 1
        dims.append(d)
        rem = max(1, rem // d)
    dims.append(max(2, rem))
    shape = tuple(dims)
    nbytes = int(np.prod(shape)) * E
    if nbytes > (512 << 20):
        continue
    axes = tuple(int(a) for a in rng.permutation(r))
    x, y = pool[:nbytes], pool[512 << 20:(512 << 20) + nbytes]
    lay, pm = vp.TensorLayout.from_shape(shape, E), vp.from_numpy_convention(axes)
    prog = vp.build_program(lay, pm)
    if os.environ.get("SWEEP_TUNE") and prog.kernel == "tile":
        prog = vp.autotune(lay, pm, candidates=int(os.environ["SWEEP_TUNE"]), src=x, dst=y, reps=3)
        # candidate index of the winner (0 = the model's choice)
        prog.metadata["won"] = next((c for c in range(16) if vp.build_program(lay, pm, candidate=c).text == prog.text), -1)
    t = bench.time_device(torch, lambda: execute_device(prog, x, out=y), 6, 2, fl, st)
    tc = bench.time_device(torch, lambda: y.copy_(x), 6, 2, fl, st)
    us, cus = sorted(t)[3] * 1e3, sorted(tc)[3] * 1e3
    m = prog.metadata
    rows.append((us and cus / us, 2 * nbytes / us / 1e3, shape, axes, E, prog.kernel, m["src_run"], m["dst_run"],
                 m["merged_dims"], m["merged_sigma"]))
    print(f"{i:3d} {rows[-1][0]:.3f} {rows[-1][1]:6.0f} GB/s {prog.kernel:5s} E={E} {shape} {axes} "
          f"runs {m['src_run']}x{m['dst_run']} T={m['tile_elems']} won={m.get('won', '-')}", flush=True)
fr = np.array([r[0] for r in rows])
print(f"\nfraction of same-size copy_: median {np.median(fr):.3f}  p10 {np.percentile(fr, 10):.3f}  "
      f"min {fr.min():.3f}  (n={len(rows)})")
print("worst:")
for r in sorted(rows)[:8]:
    print(f"  {r[0]:.3f} {r[1]:6.0f} GB/s {r[5]} E={r[4]} {r[2]} {r[3]} runs {r[6]}x{r[7]} merged {r[8]} {r[9]}")
