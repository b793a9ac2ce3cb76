"""Small cases of every kernel path for compute-sanitizer (memcheck/racecheck):
rows (whole rows, chunked rows, short predicated rows), chunked copy with
tails, bulk rows, tile kernels (aligned, shifted, ragged, congruent with VxV
W blocks, residue + address swizzle, specialised and AOT), gather, the push
and pull exchanges, and the bounded host path.  Exits non-zero on a
parity failure."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2506_03686_b200 as vp  # noqa: E402
from paper_2506_03686_b200.api import execute_device  # noqa: E402
from paper_2506_03686_b200.sharded import emulate_fused  # noqa: E402

cases = [
    ((8, 4, 256), (1, 0, 2), 4, {}),                # rows, whole rows
    ((3, 2, 64, 1001), (1, 0, 2, 3), 8, {}),        # rows, few long rows -> chunks
    ((20, 12, 66), (1, 0, 2), 8, {}),               # rows, short predicated rows
    ((5, 7, 9), (0, 1, 2), 4, {}),                  # copy (small)
    ((3, 1000003), (0, 1), 4, {}),                  # copy, chunked with a tail
    ((96, 130), (1, 0), 4, {}),                     # tile
    ((17, 9, 13, 15, 11, 27), (5, 2, 0, 4, 1, 3), 4, {}),   # tile, shifted runs, ragged
    ((17, 9, 13, 15, 11, 27), (5, 2, 0, 4, 1, 3), 4, {"jit": True}),
    ((33, 65, 129), (1, 2, 0), 2, {}),              # 2-byte words
    ((7, 5, 3), (2, 0, 1), 16, {}),                 # gather-size, 16-byte words
    ((6, 4, 1024), (1, 0, 2), 4, {}),               # rows, TMA bulk pipeline (4 KiB rows, grouped)
    ((3, 2, 5000), (1, 0, 2), 8, {}),               # rows, TMA bulk pipeline (40 KB rows, chunked)
    ((256, 512), (1, 0), 4, {}),                    # tile, congruent swizzled rows + VxV W blocks (AOT)
    ((256, 512), (1, 0), 4, {"jit": True}),         # ... specialised
    ((64, 48, 56, 8), (0, 2, 3, 1), 8, {}),         # congruent rows, 8-byte words
    ((37, 11, 45), (2, 0, 1), 4, {"jit": True}),    # residue strides mod 128 B + address swizzle
]
bad = 0
for shape, axes, E, kw in cases:
    n = int(np.prod(shape))
    prog = vp.build_program(vp.TensorLayout.from_shape(shape, E), vp.from_numpy_convention(axes), **kw)
    words = np.random.default_rng(n).integers(0, 256, size=n * E, dtype=np.uint8)
    x = torch.from_numpy(words).cuda()
    y = execute_device(prog, x)
    want = np.ascontiguousarray(np.transpose(words.view(f"V{E}").reshape(shape), axes)).reshape(-1).view(np.uint8)
    ok = np.array_equal(y.cpu().numpy().reshape(-1), want)
    bad += not ok
    print(f"{prog.kernel:6s} {shape} {axes} E={E} {kw}: {'ok' if ok else 'MISMATCH'}", flush=True)
# fused exchanges: push (two virtual ranks), pull (four)
for shape, axes, G, mode in [((8, 6, 16, 4), (2, 0, 3, 1), 2, "push"),
                             ((2,) * 16, (3, 9, 0, 7, 1, 5, 2, 11, 8, 6, 4, 10, 15, 13, 14, 12), 4, "pull")]:
    g = torch.randint(-2**31, 2**31 - 1, (int(np.prod(shape)),), dtype=torch.int32, device="cuda")
    got = torch.cat(emulate_fused(g, shape, axes, G, mode=mode))
    ok = torch.equal(got, g.view(shape).permute(axes).reshape(-1))
    bad += not ok
    print(f"exchange {mode} {shape}: {'ok' if ok else 'MISMATCH'}", flush=True)
# bounded host path
shape, axes = (16, 64, 56, 56), (0, 2, 3, 1)
h = torch.randint(-2**31, 2**31 - 1, shape, dtype=torch.int32)
prog = vp.build_program(vp.TensorLayout.from_shape(shape, 4), vp.from_numpy_convention(axes))
out, _ = vp.execute(prog, h, max_device_bytes=4 << 20)
ok = torch.equal(out.reshape(-1), h.permute(axes).reshape(-1))
bad += not ok
print(f"bounded host {shape}: {'ok' if ok else 'MISMATCH'}", flush=True)
sys.exit(1 if bad else 0)
