"""Why is the G=1 sharded step slower than the direct launch? (probe)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2506_03686_b200 import TensorLayout, build_program, from_numpy_convention, permute  # noqa: E402
from paper_2506_03686_b200.api import execute_device  # noqa: E402
from paper_2506_03686_b200.workloads import CONFIGS  # noqa: E402

wl = CONFIGS["cfg5"]
dev = torch.device("cuda", 0)
x = torch.randint(-2**62, 2**62, (wl.numel,), dtype=torch.int64, device=dev)
y = torch.empty_like(x)
prog = build_program(TensorLayout.from_shape(wl.shape, 8), from_numpy_convention(wl.axes))
x28 = x.reshape(wl.shape)


def t(f, n=5):
    for _ in range(2):
        f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        f()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


print("execute_device out=y   ", t(lambda: execute_device(prog, x, out=y)))
print("permute(x28) alloc     ", t(lambda: permute(x28, wl.axes)))
print("execute_device alloc   ", t(lambda: execute_device(prog, x)))
print("jit_state", prog.jit_state)

if os.environ.get("WITH_NCCL"):
    import torch.distributed as dist

    dist.init_process_group("nccl", device_id=dev)
    print("after nccl init: execute_device out=y", t(lambda: execute_device(prog, x, out=y)))
    print("after nccl init: permute(x28)        ", t(lambda: permute(x28, wl.axes)))
    from paper_2506_03686_b200.sharded import permute_sharded, plan_sharded
    sp = plan_sharded(wl.shape, wl.axes, 1)
    print("after nccl init: permute_sharded     ", t(lambda: permute_sharded(x, wl.shape, wl.axes, plan=sp)))
    dist.destroy_process_group()
