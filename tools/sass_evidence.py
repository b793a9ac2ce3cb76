"""Blackwell evidence from the binaries (no GPU): per-kernel counts of the
memory-movement instructions in libvpgpu.so (ahead-of-time kernels) and in
the specialised (NVRTC-equivalent, compiled here with nvcc for sm_100a)
tile kernels of the BASELINE configs.

    python tools/sass_evidence.py > profiles/sass_r2.txt

Mnemonics: LDGSTS = cp.async (global->smem, per lane), UBLKCP = cp.async.bulk
(TMA bulk copy, one thread), UTMALDG / UTMASTG = tensor-map TMA load/store,
SYNCS = mbarrier operations, LDG/STG .128 = 16-byte global accesses,
LDS/STS = shared memory, ATOM/RED = atomics (dynamic tile scheduler),
MEMBAR = fences (exchange barrier), NANOSLEEP = flag waits."""
import collections
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2506_03686_b200 import TensorLayout, _lib, build_program, from_numpy_convention  # noqa: E402
from paper_2506_03686_b200.api import emit_source  # noqa: E402
from paper_2506_03686_b200.workloads import CONFIGS  # noqa: E402

CSRC = os.path.join(ROOT, "paper_2506_03686_b200", "csrc")
KEYS = ["LDGSTS", "UBLKCP", "UTMALDG", "UTMASTG", "SYNCS", "LDG.E.128", "LDG.E.64", "LDG.E", "STG.E.128", "STG.E.64", "STG.E",
        "LDS.128", "LDS", "STS", "ATOM", "ATOMG", "RED", "MEMBAR", "NANOSLEEP", "BAR.SYNC"]


def classify(op):
    op = op.split()[0]
    for k in KEYS:
        if k in ("LDG.E", "STG.E", "LDS"):
            if op == k or (op.startswith(k + ".") and not op.startswith((k + ".128", k + ".64"))):
                return k
            continue
        if op.startswith(k):
            return k
    return None


def histogram(sass):
    """{kernel name: (instructions, Counter)} from cuobjdump -sass text."""
    out, name, cnt, tot = {}, None, None, 0
    for line in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            if name:
                out[name] = (tot, cnt)
            name, cnt, tot = m.group(1), collections.Counter(), 0
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if m and name:
            tot += 1
            k = classify(m.group(2))
            if k:
                cnt[k] += 1
    if name:
        out[name] = (tot, cnt)
    return out


def demangle(n):
    try:
        return subprocess.run(["c++filt", n], capture_output=True, text=True).stdout.strip()
    except OSError:
        return n


def show(title, hist):
    print(f"== {title}")
    for name, (tot, cnt) in sorted(hist.items()):
        body = ", ".join(f"{k} {cnt[k]}" for k in KEYS if cnt[k])
        print(f"  {demangle(name)[:110]}: {tot} instructions; {body}")


lib = _lib.LIB_PATH
show(f"libvpgpu.so (ahead-of-time kernels, {os.path.relpath(lib, ROOT)})",
     histogram(subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout))
for cfg in ("cfg1", "cfg2", "cfg3", "cfg5"):
    wl = CONFIGS[cfg]
    prog = build_program(TensorLayout.from_shape(wl.shape, wl.elem_bytes), from_numpy_convention(wl.axes))
    d = tempfile.mkdtemp()
    cu, cub = os.path.join(d, "k.cu"), os.path.join(d, "k.cubin")
    with open(cu, "w") as f:
        f.write(emit_source(prog))
    r = subprocess.run(["nvcc", "-cubin", "-gencode", "arch=compute_100a,code=sm_100a", "-std=c++17", "-I", CSRC,
                        "-Xptxas", "-v", "-o", cub, cu], capture_output=True, text=True)
    regs = re.findall(r"Used (\d+) registers", r.stderr)
    plan = [ln for ln in prog.text.splitlines() if ln.startswith(("tile elements", "vector elems"))]
    show(f"{cfg} specialised tile kernel (regs {regs[0] if regs else '?'}; {'; '.join(plan)})",
         histogram(subprocess.run(["cuobjdump", "-sass", cub], capture_output=True, text=True).stdout))
