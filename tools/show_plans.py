"""Print the planner's choice for the BASELINE configs (or given shape/axes)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_03686_b200 as vp  # noqa: E402
from paper_2506_03686_b200.workloads import CONFIGS  # noqa: E402

full = "-v" in sys.argv
for k, wl in CONFIGS.items():
    lay = vp.TensorLayout.from_shape(wl.shape, wl.elem_bytes)
    p = vp.build_program(lay, vp.from_numpy_convention(wl.axes))
    print("==", k)
    for line in p.text.splitlines():
        if full or any(w in line for w in ("phase", "pitch", "util", "tile elements", "rows:", "vector")):
            print("  ", line)
