"""Command-line front end: plan, gen, run, check, bench.

Mirrors the reference's ``vecperm`` CLI (/root/reference/pkg/src/vecperm/cli.py:
commands 196-313, flags 316-372, VPT1 tensor files 33/94-122, error lines
47-50/404-420) on the GPU path:

  python -m paper_2506_03686_b200 plan  --shape 7,32,32,3 --map 0,2,3,1
  python -m paper_2506_03686_b200 gen   --shape 64,32,32,4 --map 2,1,0,3 --out kernel.cu
  python -m paper_2506_03686_b200 run   --in input.vpt --map 0,2,3,1 --out output.vpt
  python -m paper_2506_03686_b200 check --cases 1000 --max-rank 16 --seed 7
  python -m paper_2506_03686_b200 bench --shape 4096,4096 --map 1,0

Shapes are NumPy order (outer-to-inner); ``--map`` defaults to the NumPy
convention (``--convention paper`` reads the inner-first sigma instead).
``check`` validates GPU results by properties that need no CPU permutation:
agreement with torch's own device permute (rank <= 25) and the inverse
round trip.  Errors print one ``error <code>: <message>`` line, exit 1.
"""

from __future__ import annotations

import argparse
import struct
import sys
import time

import numpy as np

from .core import LayoutError, PermutationMap, TensorLayout, from_numpy_convention, to_numpy_convention

MAGIC = 0x56505431  # "VPT1"
FAMILIES = ("all2", "pow2", "general")


class CLIError(Exception):
    def __init__(self, code: str, msg: str):
        super().__init__(msg)
        self.code = code


def parse_ints(text: str) -> tuple[int, ...]:
    try:
        return tuple(int(x) for x in text.replace(" ", "").split(",") if x != "")
    except ValueError:
        raise CLIError("bad-int-list", f"cannot parse integer list {text!r}")


def write_tensor(path: str, data: np.ndarray, layout: TensorLayout) -> None:
    """VPT1: 16-byte header (magic, elem width, rank, 0) + u32 dims outer-first + payload."""
    shape = layout.shape_outer_first()
    with open(path, "wb") as f:
        f.write(struct.pack("<4I", MAGIC, layout.elem_width, layout.rank, 0))
        f.write(struct.pack(f"<{layout.rank}I", *shape))
        f.write(np.ascontiguousarray(data).reshape(-1).view(np.uint8).tobytes())


def read_tensor(path: str) -> tuple[TensorLayout, np.ndarray]:
    with open(path, "rb") as f:
        head = f.read(16)
        if len(head) != 16:
            raise CLIError("bad-tensor-file", f"{path}: truncated header")
        magic, elem, rank, _ = struct.unpack("<4I", head)
        if magic != MAGIC:
            raise CLIError("bad-tensor-file", f"{path}: bad magic {magic:#x}")
        raw = f.read(4 * rank)
        if len(raw) != 4 * rank:
            raise CLIError("bad-tensor-file", f"{path}: truncated dims")
        try:
            layout = TensorLayout.from_shape(struct.unpack(f"<{rank}I", raw), elem)
        except LayoutError as e:
            raise CLIError("bad-tensor-file", f"{path}: {e}")
        payload = np.frombuffer(f.read(), dtype=np.uint8)
    if payload.size != layout.num_elements * elem:
        raise CLIError("bad-tensor-file", f"{path}: payload size mismatch")
    return layout, payload


def job(args) -> tuple[TensorLayout, PermutationMap]:
    if getattr(args, "in_path", None):
        layout, _ = read_tensor(args.in_path)
    else:
        if not args.shape:
            raise CLIError("missing-shape", "--shape is required")
        try:
            layout = TensorLayout.from_shape(parse_ints(args.shape), args.elem)
        except LayoutError as e:
            raise CLIError("bad-shape", str(e))
    if args.map is None:
        return layout, PermutationMap(tuple(range(layout.rank)))
    entries = parse_ints(args.map)
    if len(entries) != layout.rank:
        raise CLIError("bad-map", f"map rank {len(entries)} != shape rank {layout.rank}")
    try:
        pm = from_numpy_convention(entries) if args.convention == "numpy" else PermutationMap(tuple(reversed(entries)))
    except LayoutError as e:
        raise CLIError("bad-map", str(e))
    return layout, pm


def _program(args, layout, pmap):
    from .api import build_program

    try:
        return build_program(layout, pmap, merge=not args.no_merge)
    except LayoutError as e:
        raise CLIError("bad-plan", str(e))


def cmd_plan(args) -> int:
    layout, pmap = job(args)
    prog = _program(args, layout, pmap)
    print(f"shape (outer->inner): {layout.shape_outer_first()}")
    print(f"map (numpy axes): {to_numpy_convention(pmap)}  (sigma, inner-first): {pmap.sigma}")
    print(prog.text)
    return 0


def cmd_gen(args) -> int:
    from .api import emit_source

    layout, pmap = job(args)
    prog = _program(args, layout, pmap)
    try:
        src = emit_source(prog)
    except LayoutError as e:
        raise CLIError("no-source", f"{prog.kernel} plans run a fixed kernel: {e}")
    if args.out:
        with open(args.out, "w") as f:
            f.write(src)
    else:
        sys.stdout.write(src)
    return 0


def _device():
    import torch

    if not torch.cuda.is_available():
        raise CLIError("no-gpu", "no CUDA device (the permutation runs only on the GPU)")
    return torch


def cmd_run(args) -> int:
    from .api import execute

    layout, pmap = job(args)
    if args.in_path:
        _, payload = read_tensor(args.in_path)
    else:
        rng = np.random.default_rng(args.seed)
        payload = rng.integers(0, 256, size=layout.num_elements * layout.elem_width, dtype=np.uint8)
    prog = _program(args, layout, pmap)
    torch = _device()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    # host buffer in, host buffer out (pipelined; streamed through bounded
    # device scratch when the tensor does not fit, or --max-device-bytes)
    out, _ = execute(prog, np.ascontiguousarray(payload).view(np.uint8),
                     max_device_bytes=args.max_device_bytes)
    dt = time.perf_counter() - t0
    out = np.ascontiguousarray(out).view(np.uint8).reshape(-1)
    if args.out:
        from .core import permuted_layout

        write_tensor(args.out, out, permuted_layout(layout, pmap))
    if args.stats:
        print(f"kernel: {prog.kernel}")
        print(f"elements: {layout.num_elements}")
        print(f"bytes_moved: {prog.algorithmic_bytes}")
        print(f"wall_s: {dt:.6f} (host to host, includes transfers; see bench)")
    return 0


def sample_case(rng, max_rank, max_elems):
    """The reference campaign's sampler semantics (cli.py:129-149)."""
    family = FAMILIES[int(rng.integers(0, 3))]
    rank = int(rng.integers(2, max_rank + 1))
    dims = (2, 2)
    for _ in range(64):
        if family == "all2":
            dims = (2,) * rank
        elif family == "pow2":
            dims = tuple(int(2 ** rng.integers(0, 6)) for _ in range(rank))
        else:
            dims = tuple(int(rng.integers(1, 10)) for _ in range(rank))
        if int(np.prod(dims)) <= max_elems:
            break
        rank = max(2, rank - 1)
    sigma = tuple(int(x) for x in rng.permutation(len(dims)))
    elem = (4, 8)[int(rng.integers(0, 2))]
    return family, TensorLayout(dims, elem), PermutationMap(sigma)


def run_campaign(cases, max_rank=16, seed=0, max_elems=1 << 16, progress=None) -> dict:
    """Randomized GPU validation by device-side properties (no CPU oracle):
    torch's permute for rank <= 25 and the inverse round trip for all."""
    torch = _device()
    from .api import build_program, execute_device
    from .core import permuted_layout

    rng = np.random.default_rng(seed)
    mismatches, per_family = [], {f: 0 for f in FAMILIES}
    for i in range(cases):
        family, layout, pmap = sample_case(rng, max_rank, max_elems)
        per_family[family] += 1
        n = layout.num_elements
        word = torch.int32 if layout.elem_width == 4 else torch.int64
        x = torch.randint(-2**31, 2**31 - 1, (n,), dtype=word, device="cuda")
        y = execute_device(build_program(layout, pmap), x)
        back = execute_device(build_program(permuted_layout(layout, pmap), pmap.inverse()), y)
        ok = torch.equal(back.reshape(-1), x)
        if ok and layout.rank <= 25:
            ok = torch.equal(y.reshape(-1), x.reshape(layout.shape_outer_first())
                             .permute(to_numpy_convention(pmap)).contiguous().reshape(-1))
        if not ok:
            mismatches.append({"shape": layout.shape_outer_first(), "sigma": pmap.sigma})
        if progress and (i + 1) % progress == 0:
            print(f"  {i + 1}/{cases} cases done", flush=True)
    return {"cases": cases, "passed": cases - len(mismatches), "mismatches": mismatches, "per_family": per_family}


def cmd_check(args) -> int:
    summary = run_campaign(args.cases, args.max_rank, args.seed, args.max_elems, progress=args.progress)
    print(f"passed {summary['passed']}/{summary['cases']}  families {summary['per_family']}")
    for m in summary["mismatches"][:10]:
        print(f"MISMATCH shape={m['shape']} sigma={m['sigma']}")
    return 0 if not summary["mismatches"] else 1


def cmd_bench(args) -> int:
    torch = _device()
    from .api import execute_device

    layout, pmap = job(args)
    prog = _program(args, layout, pmap)
    nbytes = prog.nbytes
    x = torch.randint(0, 255, (nbytes,), dtype=torch.uint8, device="cuda")
    y = torch.empty_like(x)
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    fl_w = torch.empty(max(2 * l2, 256 << 20) // 4, dtype=torch.float32, device="cuda")
    fl_r = torch.zeros_like(fl_w)
    times = []
    for it in range(args.warmup + args.steps):
        fl_w.fill_(1.0)
        fl_r.sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        execute_device(prog, x, out=y)
        b.record()
        if it >= args.warmup:
            times.append((a, b))
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in times)[len(times) // 2]
    print(f"kernel {prog.kernel}: median {ms * 1e3:.1f} us, {prog.algorithmic_bytes / ms / 1e6:.0f} GB/s effective "
          f"(read+write, L2 flushed before each launch)")
    return 0


def build_parser():
    ap = argparse.ArgumentParser(prog="python -m paper_2506_03686_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)

    def common(p):
        p.add_argument("--shape", default=None)
        p.add_argument("--map", default=None)
        p.add_argument("--convention", choices=("numpy", "paper"), default="numpy")
        p.add_argument("--elem", type=int, default=4)
        p.add_argument("--no-merge", action="store_true")
        p.add_argument("--seed", type=int, default=0)

    p = sub.add_parser("plan")
    common(p)
    p = sub.add_parser("gen")
    common(p)
    p.add_argument("--out", default=None)
    p = sub.add_parser("run")
    common(p)
    p.add_argument("--in", dest="in_path", default=None)
    p.add_argument("--out", default=None)
    p.add_argument("--stats", action="store_true")
    p.add_argument("--max-device-bytes", type=int, default=None,
                   help="stream through at most this much device scratch")
    p = sub.add_parser("check")
    p.add_argument("--cases", type=int, default=1000)
    p.add_argument("--max-rank", type=int, default=16)
    p.add_argument("--max-elems", type=int, default=1 << 16)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--progress", type=int, default=0)
    p = sub.add_parser("bench")
    common(p)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return {"plan": cmd_plan, "gen": cmd_gen, "run": cmd_run, "check": cmd_check, "bench": cmd_bench}[args.cmd](args)
    except CLIError as e:
        print(f"error {e.code}: {e}", file=sys.stderr)
        return 1
    except LayoutError as e:
        print(f"error layout: {e}", file=sys.stderr)
        return 1
