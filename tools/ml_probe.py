"""Common ML layout changes (attention head splits/merges, NCHW<->NHWC,
image channel moves, batched transposes) in f32 / bf16 / u8 against a
same-size copy_: flushed means of 20 launches, the planner's choice."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_03686_b200 as vp  # noqa: E402
from paper_2506_03686_b200.api import execute_device  # noqa: E402

CASES = [
    ("attn split  (B,S,H,D)->(B,H,S,D)", (8, 2048, 32, 128), (0, 2, 1, 3)),
    ("attn split  small head", (16, 1024, 12, 64), (0, 2, 1, 3)),
    ("attn K^T    (B,H,S,D)->(B,H,D,S)", (8, 32, 2048, 128), (0, 1, 3, 2)),
    ("NCHW->NHWC  resnet", (64, 256, 56, 56), (0, 2, 3, 1)),
    ("NHWC->NCHW  resnet", (64, 56, 56, 256), (0, 3, 1, 2)),
    ("NCHW->NHWC  7x7", (64, 2048, 7, 7), (0, 2, 3, 1)),
    ("image CHW->HWC", (32, 3, 512, 512), (0, 2, 3, 1)),
    ("image HWC->CHW", (32, 512, 512, 3), (0, 3, 1, 2)),
    ("batched 2-D transpose", (64, 1024, 1000), (0, 2, 1)),
    ("MoE (E,T,D)->(T,E,D)", (64, 4096, 1024), (1, 0, 2)),
    ("conv weight OIHW->HWIO", (512, 256, 3, 3), (2, 3, 1, 0)),
]
dev = torch.device("cuda", 0)
fl = bench.Flusher(torch, dev)
st = torch.cuda.current_stream()
for E, name in ((4, "f32"), (2, "bf16"), (1, "u8")):
    for label, shape, axes in CASES:
        n = int(np.prod(shape)) * E
        if n > (1 << 30):
            continue
        x = torch.randint(0, 255, (n,), dtype=torch.uint8, device=dev)
        y = torch.empty_like(x)
        p = vp.build_program(vp.TensorLayout.from_shape(shape, E), vp.from_numpy_convention(axes))
        t = np.mean(bench.time_device(torch, lambda: execute_device(p, x, out=y), 20, 3, fl, st)) * 1e3
        tc = np.mean(bench.time_device(torch, lambda: y.copy_(x), 20, 3, fl, st)) * 1e3
        vec = [ln.split(":", 1)[1].strip()[:60] for ln in p.text.splitlines()
               if ln.startswith("vector") or ln.startswith("rows:")][:1]
        print(f"{name:4s} {label:34s} {str(shape):22s} {n / 2**20:7.1f} MiB {p.kernel:5s} {t:8.2f} us "
              f"{tc / t:.3f} of copy_ {2 * n / t / 1e3:6.0f} GB/s  {vec}", flush=True)
        del x, y
