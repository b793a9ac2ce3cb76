"""Emit a config's specialised tile kernel (emit_source), compile it for
sm_100a with nvcc here (no GPU needed) and print the static SASS opcode
histogram plus register count -- a CPU-side check of the per-element
instruction cost before spending GPU time.

    python tools/sass_count.py cfg3 [cfg2 ...]
"""
import collections
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2506_03686_b200 import TensorLayout, build_program, from_numpy_convention  # noqa: E402
from paper_2506_03686_b200.api import emit_source  # noqa: E402
from paper_2506_03686_b200.workloads import CONFIGS  # noqa: E402

CSRC = os.path.join(ROOT, "paper_2506_03686_b200", "csrc")


def sass_of(src):
    d = tempfile.mkdtemp()
    cu = os.path.join(d, "k.cu")
    with open(cu, "w") as f:
        f.write(src)
    cub = os.path.join(d, "k.cubin")
    r = subprocess.run(["nvcc", "-cubin", "-gencode", "arch=compute_100a,code=sm_100a", "-std=c++17", "-I", CSRC,
                        "-Xptxas", "-v", "-o", cub, cu], capture_output=True, text=True)
    if r.returncode:
        raise SystemExit(r.stderr)
    regs = re.findall(r"Used (\d+) registers", r.stderr)
    sass = subprocess.run(["cuobjdump", "-sass", cub], capture_output=True, text=True).stdout
    return sass, regs


for cfg in sys.argv[1:] or ["cfg3"]:
    wl = CONFIGS[cfg]
    prog = build_program(TensorLayout.from_shape(wl.shape, wl.elem_bytes), from_numpy_convention(wl.axes))
    sass, regs = sass_of(emit_source(prog))
    ops = collections.Counter()
    for line in sass.splitlines():
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m:
            ops[m.group(2)] += 1
    tot = sum(ops.values())
    print(f"{cfg}: {tot} static SASS instructions, regs {regs}; "
          + ", ".join(f"{k} {v}" for k, v in ops.most_common(14)))
