import sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_2506_03686_b200 as vp
from paper_2506_03686_b200.api import execute_device
shape, axes, E = (1024, 1024), (1, 0), 4
p = vp.build_program(vp.TensorLayout.from_shape(shape, E), vp.from_numpy_convention(axes))
print(p.jit_state, p.text)
x = torch.randint(0, 255, (1024*1024*4,), dtype=torch.uint8, device="cuda")
y = torch.empty_like(x)
for _ in range(3): execute_device(p, x, out=y)
torch.cuda.synchronize()
