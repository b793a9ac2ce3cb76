"""SM-kernel copy ceiling vs the copy engine: identity permutation through
libvpgpu's copy_kernel (16-byte vectors, grid-stride) and torch's copy_
(cudaMemcpy D2D) of the cfg5 byte count, flushed single launches."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_03686_b200 as vp  # noqa: E402
from paper_2506_03686_b200.api import execute_device  # noqa: E402

dev = torch.device("cuda", 0)
fl = bench.Flusher(torch, dev)
st = torch.cuda.current_stream()
for nbytes in (1 << 31, 1 << 30, 1 << 28):
    x = torch.randint(0, 255, (nbytes,), dtype=torch.uint8, device=dev)
    y = torch.empty_like(x)
    prog = vp.build_program(vp.TensorLayout.from_shape((nbytes // 8,), 8), vp.from_numpy_convention((0,)))
    t1 = bench.time_device(torch, lambda: execute_device(prog, x, out=y), 10, 3, fl, st)
    t2 = bench.time_device(torch, lambda: y.copy_(x), 10, 3, fl, st)
    m1, m2 = sorted(t1)[5] * 1e3, sorted(t2)[5] * 1e3
    print(f"{nbytes >> 20} MiB: copy_kernel ({prog.kernel}) {m1:8.1f} us {2*nbytes/m1/1e3:6.0f} GB/s | "
          f"torch copy_ {m2:8.1f} us {2*nbytes/m2/1e3:6.0f} GB/s", flush=True)
