"""Planner calibration data: for random permutations (the perf_sweep.py
generator, 32-512 MiB), every distinct tile candidate of the cost model at
three staging budgets is timed (flushed launches, mean of 10) against a
same-size copy_, with the model's terms (describe(): geometry cost, sector
efficiencies, walk cost, lane utilisation) and the plan's layout (runs,
tile, pitch, stages, smem, tiles).  One JSON line per candidate to stdout.

    python tools/cand_data.py N seed > gpurun_out/cand_data.jsonl
"""
import json
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_03686_b200 as vp  # noqa: E402
from paper_2506_03686_b200.api import execute_device  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 30
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 21
rng = np.random.default_rng(seed)
dev = torch.device("cuda", 0)
fl = bench.Flusher(torch, dev)
st = torch.cuda.current_stream()
HI = 512 << 20
pool = torch.empty(2 * HI, dtype=torch.uint8, device=dev)


def num(pat, text, cast=float, default=None):
    m = re.search(pat, text)
    return cast(m.group(1)) if m else default


def features(p):
    t = p.text
    return {
        "Ls": p.metadata["src_run"], "Ld": p.metadata["dst_run"], "T": p.metadata["tile_elems"],
        "pitch": p.metadata["smem_pitch"], "smem": p.metadata["smem_bytes"], "threads": p.metadata["threads"],
        "tiles": p.metadata["num_tiles"],
        "buffers": num(r"buffers: (\d+)", t, int),
        "util": num(r"lane utilisation \(R\*W\): ([0-9.]+)", t),
        "geom": num(r"cost model: geometry ([0-9.]+)", t),
        "eff_s": num(r"sector efficiency src ([0-9.]+)", t),
        "eff_d": num(r"dst ([0-9.]+)\), walk", t),
        "walk": num(r"walk ([0-9.]+) per element", t),
        "vec": re.search(r"vector elems: (.*)", t).group(1) if "vector elems" in t else "",
        "ragged": re.search(r"ragged boundary dims: (.*)", t).group(1) if "ragged boundary" in t else "",
    }


def shapes():
    if "CAND_WORDS" not in os.environ:
        yield (17, 9, 13, 15, 11, 27), (5, 2, 0, 4, 1, 3), 4
        yield (8, 2, 5, 158, 37, 143), (2, 1, 0, 5, 4, 3), 4
    for _ in range(N):
        E = int(rng.choice([int(w) for w in os.environ.get("CAND_WORDS", "4,8").split(",")]))
        target = int(rng.choice([32, 64, 128, 256, 512])) << 20
        r = int(rng.integers(2, 8))
        n = target // E
        dims, rem = [], n
        for k in range(r - 1):
            h = max(2, int(round(rem ** (1.0 / (r - k)) * rng.uniform(0.5, 2.0))))
            d = int(rng.integers(2, h + 1))
            if rng.random() < 0.5:
                d = d | 1
            dims.append(d)
            rem = max(1, rem // d)
        dims.append(max(2, rem))
        yield tuple(dims), tuple(int(a) for a in rng.permutation(r)), E


for si, (shape, axes, E) in enumerate(shapes()):
    nbytes = int(np.prod(shape)) * E
    if nbytes > HI:
        continue
    lay, pm = vp.TensorLayout.from_shape(shape, E), vp.from_numpy_convention(axes)
    os.environ.pop("VPG_TILE_BUDGET", None)
    vp.program_cache_clear()
    default = vp.build_program(lay, pm)
    if default.kernel != "tile":
        continue
    x, y = pool[:nbytes], pool[HI:HI + nbytes]
    tc = float(np.mean(bench.time_device(torch, lambda: y.copy_(x), 10, 2, fl, st))) * 1e3
    seen = {}
    cands = [("default", None, default)]
    for budget in (24576, 32768, 49152):
        os.environ["VPG_TILE_BUDGET"] = str(budget)
        for k in range(6):
            vp.program_cache_clear()
            try:
                p = vp.build_program(lay, pm, candidate=k)
            except vp.LayoutError:
                break
            cands.append((budget, k, p))
    os.environ.pop("VPG_TILE_BUDGET", None)
    for budget, k, p in cands:
        key = p.text.split("specialised")[0]
        if key in seen:
            if budget == "default":
                continue
            continue
        seen[key] = True
        t = float(np.mean(bench.time_device(torch, lambda: execute_device(p, x, out=y), 10, 2, fl, st))) * 1e3
        rec = {"shape_id": si, "shape": shape, "axes": axes, "E": E, "bytes": nbytes, "budget": budget, "cand": k,
               "us": round(t, 3), "copy_us": round(tc, 3), "frac_copy": round(tc / t, 4),
               "is_default": budget == "default"}
        rec.update(features(p))
        print(json.dumps(rec), flush=True)
