"""Run one permutation a few times (for ncu / sanitizers):
    python tools/run_shape.py "(17, 20, 18, 11, 6, 664)" "(5, 4, 3, 1, 0, 2)" 2 [iters]"""
import ast
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2506_03686_b200 as vp  # noqa: E402
from paper_2506_03686_b200.api import execute_device  # noqa: E402

shape, axes, E = ast.literal_eval(sys.argv[1]), ast.literal_eval(sys.argv[2]), int(sys.argv[3])
iters = int(sys.argv[4]) if len(sys.argv) > 4 else 3
p = vp.build_program(vp.TensorLayout.from_shape(shape, E), vp.from_numpy_convention(axes))
print(p.text, flush=True)
n = int(np.prod(shape)) * E
x = torch.randint(0, 255, (n,), dtype=torch.uint8, device="cuda")
y = torch.empty_like(x)
for _ in range(iters):
    execute_device(p, x, out=y)
torch.cuda.synchronize()
print("done")
