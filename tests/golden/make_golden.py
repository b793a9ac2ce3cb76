"""Generate tests/golden/golden.json FROM THE REFERENCE ITSELF (run in the
build container, where /root/reference exists; the GPU box only reads the
committed JSON).

Every case is run through the reference's oracle ``vecperm.core.naive_permute``
(/root/reference/pkg/src/vecperm/core.py:192-204) and its planner's
``merge_dimensions`` (planner.py:211-241).  We store:

* the case: numpy shape/axes, inner-first dims/sigma (via the reference's
  ``from_numpy_convention``, core.py:144-149), element width;
* ``merged_dims`` / ``merged_sigma`` from the reference's merge;
* ``sha256`` of the reference output for the deterministic input pattern
  ``golden_pattern`` below (distinct words at every position, full-width --
  the 8-byte pattern sets the high 32 bits, closing SURVEY.md §4's gap);
* the full output words for small cases (``out`` when N <= 512).

Case families:
* known answers of the reference tests (test_core.py:93-100, 147-151);
* the paper shape (7,32,32,3) / (0,2,3,1) (test_cli.py:69-83);
* SURVEY Appendix A edge cases and the merge known answers
  (test_planner.py:24-61);
* the N = 2**20 transpose (test_acceptance.py:35-44);
* the reference's randomized campaign: the exact 1000 cases the reference's
  ``run_campaign(1000, max_rank=16, seed=2024, max_elems=1<<16)`` draws
  (test_acceptance.py:25-33; cli.py:129-189), reproduced by calling the
  reference's own ``sample_case`` with the same rng consumption;
* a ragged-destination sweep (test_acceptance.py:250-274 shapes);
* full-size BASELINE configs: sha256 of input and output bytes, output from
  the reference's emitted AVX-512 kernel (oracle/_ref), cross-checked here
  against the reference's naive_permute (cfg1-3) and numpy transpose (all).

Usage: python tests/golden/make_golden.py [--skip-full]
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"
sys.dont_write_bytecode = True
sys.path.insert(0, REF_SRC)
sys.path.insert(0, REPO)

from vecperm.cli import sample_case  # noqa: E402
from vecperm.core import (  # noqa: E402
    PermutationMap,
    TensorLayout,
    from_numpy_convention,
    naive_permute,
    to_numpy_convention,
)
from vecperm.planner import merge_dimensions  # noqa: E402

from tests.golden.pattern import golden_pattern  # noqa: E402


def case_entry(name, dims_inner, sigma_inner, elem, family, keep_out_max=512):
    lay = TensorLayout(tuple(dims_inner), elem)
    pm = PermutationMap(tuple(sigma_inner))
    n = lay.num_elements
    data = golden_pattern(n, elem)
    out = naive_permute(data, lay, pm)
    ml, mp = merge_dimensions(lay, pm)
    e = {
        "name": name,
        "family": family,
        "shape": list(lay.shape_outer_first()),
        "axes": list(to_numpy_convention(pm)),
        "dims": list(lay.dims),
        "sigma": list(pm.sigma),
        "elem": elem,
        "n": n,
        "merged_dims": list(ml.dims),
        "merged_sigma": list(mp.sigma),
        "sha256": hashlib.sha256(out.tobytes()).hexdigest(),
    }
    if n <= keep_out_max:
        e["out"] = [int(v) for v in out]
    return e


def numpy_case(name, shape, axes, elem, family):
    pm = from_numpy_convention(axes)
    return case_entry(name, tuple(reversed(shape)), pm.sigma, elem, family)


def small_cases():
    cases = []
    # known answers (test_core.py:147-151, 93-100)
    cases.append(numpy_case("ka_2x3_transpose", (2, 3), (1, 0), 4, "known"))
    cases.append(case_entry("ka_bitrev_2x2x2", (2, 2, 2), (2, 1, 0), 4, "known"))
    cases.append(numpy_case("ka_identity_2x5x3", (2, 5, 3), (0, 1, 2), 4, "known"))
    cases.append(case_entry("ka_elem8_3x4x2", (3, 4, 2), (2, 0, 1), 8, "known"))
    # paper shape (test_cli.py:69-83)
    cases.append(numpy_case("paper_7x32x32x3", (7, 32, 32, 3), (0, 2, 3, 1), 4, "paper"))
    cases.append(numpy_case("paper_7x32x32x3_e8", (7, 32, 32, 3), (0, 2, 3, 1), 8, "paper"))
    # merge known answers (test_planner.py:24-61), inner-first
    cases.append(case_entry("merge_3_5_7", (3, 5, 7), (2, 0, 1), 4, "merge"))
    cases.append(case_entry("merge_9_8_4", (9, 8, 4), (2, 0, 1), 4, "merge"))
    cases.append(case_entry("merge_identity", (3, 4, 5), (0, 1, 2), 4, "merge"))
    cases.append(case_entry("merge_size1", (3, 1, 5, 2), (3, 0, 1, 2), 4, "merge"))
    # SURVEY Appendix A edge cases (numpy convention)
    for shape, axes in [((64, 32, 27), (1, 0, 2)), ((64, 32, 3), (1, 0, 2)), ((5, 7, 9), (0, 1, 2)),
                        ((1, 8, 1, 16), (2, 3, 0, 1)), ((1, 1), (1, 0)), ((6, 5, 7, 3), (1, 0, 2, 3)),
                        ((1,), (0,)), ((7,), (0,)), ((3, 1), (1, 0))]:
        for elem in (4, 8):
            nm = "edge_" + "x".join(map(str, shape)) + "_" + "".join(map(str, axes)) + f"_e{elem}"
            cases.append(numpy_case(nm, shape, axes, elem, "edge"))
    # N = 2**20 transpose (test_acceptance.py:35-44)
    cases.append(case_entry("full_1024x1024", (1024, 1024), (1, 0), 4, "fullsize"))
    # tail-store safety shapes (test_acceptance.py:241-248)
    cases.append(case_entry("tail_8x5", (8, 5), (1, 0), 4, "ragged"))
    return cases


def campaign_cases(count=1000, seed=2024, max_rank=16, max_elems=1 << 16):
    """The reference campaign's cases, same rng consumption (cli.py:152-172)."""
    rng = np.random.default_rng(seed)
    out = []
    for i in range(count):
        family, layout, pmap, machine = sample_case(rng, max_rank, max_elems)
        # consume the data draw exactly as run_campaign does (cli.py:168-170)
        rng.integers(0, 2**32 - 1, size=layout.num_elements, dtype=np.uint32)
        e = case_entry(f"campaign_{i:04d}", layout.dims, pmap.sigma, layout.elem_width,
                       "campaign_" + family)
        e["w"] = machine.lanes
        out.append(e)
    return out


def ragged_sweep(seed=57, tries=60):
    """Shapes of the ragged-destination sweep (test_acceptance.py:250-274)."""
    rng = np.random.default_rng(seed)
    out = []
    for t in range(tries):
        rank = int(rng.integers(1, 5))
        dims = tuple(int(rng.integers(1, 10)) for _ in range(rank))
        n = int(np.prod(dims))
        if n > 4000:
            continue
        sigma = tuple(int(x) for x in rng.permutation(rank))
        for elem in (4, 8):
            out.append(case_entry(f"ragged_{t:02d}_e{elem}", dims, sigma, elem, "ragged"))
    return out


def full_configs():
    from oracle.refkernels import RefKernel
    from paper_2506_03686_b200.workloads import CONFIGS, make_input

    res = {}
    for key, wl in CONFIGS.items():
        x = make_input(wl)
        rk = RefKernel(key, "x86-avx")
        out = rk(x)
        want = np.ascontiguousarray(np.transpose(x, wl.axes)).reshape(-1).view(np.uint8)
        assert np.array_equal(out, want), key
        if wl.numel <= 1 << 24:
            lay = TensorLayout(tuple(reversed(wl.shape)), wl.elem_bytes)
            ref = naive_permute(x.reshape(-1).view(lay.dtype), lay, from_numpy_convention(wl.axes))
            assert np.array_equal(ref.view(np.uint8), out), key
            checked = "reference naive_permute + reference AVX-512 kernel + numpy transpose"
        else:
            checked = "reference AVX-512 kernel + numpy transpose"
        res[key] = {
            "shape": list(wl.shape),
            "axes": list(wl.axes),
            "dtype": wl.dtype,
            "seed": 0,
            "input_sha256": hashlib.sha256(x.tobytes()).hexdigest(),
            "output_sha256": hashlib.sha256(out.tobytes()).hexdigest(),
            "checked_with": checked,
        }
        print(f"[golden] {key} done", flush=True)
        del x, out, want
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-full", action="store_true")
    args = ap.parse_args()
    path = os.path.join(HERE, "golden.json")
    prev = {}
    if os.path.exists(path):
        with open(path) as f:
            prev = json.load(f)
    doc = {
        "generator": "tests/golden/make_golden.py (reference vecperm at /root/reference/pkg)",
        "pattern": "tests/golden/pattern.py:golden_pattern",
        "cases": small_cases() + ragged_sweep() + campaign_cases(),
    }
    doc["full_configs"] = prev.get("full_configs", {}) if args.skip_full else full_configs()
    with open(path, "w") as f:
        json.dump(doc, f, separators=(",", ":"))
    print(f"[golden] {len(doc['cases'])} cases -> {path}")


if __name__ == "__main__":
    main()
