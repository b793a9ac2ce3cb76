"""Quick correctness check of the bulk (TMA + mbarrier) tile path, AOT and JIT."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2506_03686_b200 import TensorLayout, build_program, from_numpy_convention  # noqa: E402
from paper_2506_03686_b200.api import execute_device  # noqa: E402

for shape, axes, E in [((256, 384), (1, 0), 4), ((64, 48), (1, 0), 4), ((8, 24, 20, 12), (0, 2, 3, 1), 4),
                       ((2,) * 16, tuple(range(15, -1, -1)), 8), ((4096, 4096), (1, 0), 4)]:
    for jit in (False, True):
        prog = build_program(TensorLayout.from_shape(shape, E), from_numpy_convention(axes), force="tile", jit=jit)
        dt = torch.int32 if E == 4 else torch.int64
        x = torch.randint(-2**30, 2**30, shape, dtype=dt, device="cuda")
        y = execute_device(prog, x)
        torch.cuda.synchronize()
        ok = torch.equal(y, x.permute(axes).contiguous())
        print(shape, axes, "jit" if jit else "aot", "bulk" if "TMA bulk" in prog.text else "-", ok, prog.jit_state,
              flush=True)
