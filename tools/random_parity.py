"""Random-shape parity campaign on the GPU against torch's own permute:
    python tools/random_parity.py N seed "1,2"   (word sizes)
Shapes of 0.25-64 MiB, ranks 2-7, many extents multiples of 2/4/8 (the gather
block widths) and many odd; specialised and ahead-of-time kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2506_03686_b200 as vp  # noqa: E402
from paper_2506_03686_b200.api import execute_device  # noqa: E402

N, seed = int(sys.argv[1]), int(sys.argv[2])
words = [int(w) for w in sys.argv[3].split(",")]
rng = np.random.default_rng(seed)
dt = {1: torch.uint8, 2: torch.int16, 4: torch.int32, 8: torch.int64}
modes = {}
bad = 0
for it in range(N):
    E = int(rng.choice(words))
    target = int(2 ** rng.uniform(18, 26)) // E
    r = int(rng.integers(2, 8))
    dims, rem = [], target
    for k in range(r - 1):
        hi = max(2, int(round(rem ** (1.0 / (r - k)) * rng.uniform(0.5, 2.0))))
        d = int(rng.integers(2, hi + 1))
        u = rng.random()
        if u < 0.25:
            d |= 1
        elif u < 0.6:
            d = max(2, d // int(rng.choice([2, 4, 8])) * int(rng.choice([2, 4, 8])))
        dims.append(d)
        rem = max(1, rem // d)
    dims.append(max(2, rem))
    shape = tuple(dims)
    axes = tuple(int(a) for a in rng.permutation(r))
    n = int(np.prod(shape))
    x = torch.randint(0, 255, (n * E,), dtype=torch.uint8, device="cuda")
    want = x.view(dt[E]).view(shape).permute(axes).reshape(-1)
    for jit in (True, False):
        p = vp.build_program(vp.TensorLayout.from_shape(shape, E), vp.from_numpy_convention(axes), jit=jit)
        got = execute_device(p, x).view(dt[E]).view(-1)
        vec = [ln for ln in p.text.splitlines() if ln.startswith("vector")]
        key = (p.kernel, E, vec[0][14:].split("(")[1][:22] if vec and "(" in vec[0] else (vec[0][14:30] if vec else ""))
        modes[key] = modes.get(key, 0) + 1
        if not torch.equal(got, want):
            bad += 1
            print("MISMATCH", shape, axes, E, jit, p.text, flush=True)
print(f"{N} shapes x 2 kernels, mismatches: {bad}")
for k, v in sorted(modes.items(), key=lambda kv: -kv[1]):
    print(f"  {v:5d}  {k}")
