"""Pin the CPU oracle (test infrastructure) to the reference itself.

Both restatements of the reference oracle -- numpy (oracle.naive_permute_np)
and C (oracle/naive_permute.c) -- must reproduce the golden vectors the
reference generated (tests/golden/make_golden.py: vecperm.core.naive_permute
on every case, including the exact 1000 cases of the reference's randomized
campaign).  Mirrors the reference's own oracle tests
(/root/reference/pkg/tests/test_core.py:93-221).
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle
from tests.golden.pattern import golden_pattern
from tests.helpers import golden, sha256


def _word(elem):
    return {4: np.uint32, 8: np.uint64}[elem]


def test_golden_file_shape():
    g = golden()
    fams = {c["family"] for c in g["cases"]}
    assert {"known", "paper", "merge", "edge", "ragged", "fullsize"} <= fams
    assert sum(c["family"].startswith("campaign_") for c in g["cases"]) == 1000
    assert set(g["full_configs"]) == {"cfg1", "cfg2", "cfg3", "cfg4", "cfg5"}


def test_c_oracle_all_golden_cases():
    bad = []
    for c in golden()["cases"]:
        data = golden_pattern(c["n"], c["elem"])
        out = oracle.naive_permute_c(data, c["dims"], c["sigma"])
        if sha256(out) != c["sha256"]:
            bad.append(c["name"])
        if "out" in c:
            assert out.view(_word(c["elem"])).tolist() == c["out"], c["name"]
    assert not bad, bad[:5]


def test_numpy_oracle_small_golden_cases():
    for c in golden()["cases"]:
        if c["n"] > 4096:
            continue
        data = golden_pattern(c["n"], c["elem"])
        out = oracle.naive_permute_np(data, c["dims"], c["sigma"])
        assert sha256(out) == c["sha256"], c["name"]


def test_known_answers():
    # test_core.py:147-151 and :93-100
    assert oracle.naive_permute_c(np.arange(6, dtype=np.uint32), (3, 2), (1, 0)).tolist() == [0, 3, 1, 4, 2, 5]
    assert oracle.bijection_c((2, 2, 2), (2, 1, 0), np.arange(8)).tolist() == [0, 4, 2, 6, 1, 5, 3, 7]


def test_numpy_axes_conversion_matches_transpose():
    rng = np.random.default_rng(2)
    for _ in range(30):
        rank = int(rng.integers(1, 6))
        shape = tuple(int(rng.integers(1, 5)) for _ in range(rank))
        axes = tuple(int(a) for a in rng.permutation(rank))
        x = rng.integers(0, 2**32 - 1, size=shape, dtype=np.uint32)
        dims, sigma = oracle.from_numpy_axes(shape, axes)
        want = np.ascontiguousarray(np.transpose(x, axes)).reshape(-1)
        assert np.array_equal(oracle.naive_permute_c(x.reshape(-1), dims, sigma), want)
        assert np.array_equal(oracle.naive_permute_np(x.reshape(-1), dims, sigma), want)


@pytest.mark.parametrize("elem", [1, 2, 16])
def test_c_oracle_superset_widths(elem):
    """1/2/16-byte words (beyond the reference's 4/8) agree with numpy transpose."""
    rng = np.random.default_rng(elem)
    for _ in range(20):
        rank = int(rng.integers(1, 5))
        shape = tuple(int(rng.integers(1, 6)) for _ in range(rank))
        axes = tuple(int(a) for a in rng.permutation(rank))
        n = int(np.prod(shape))
        raw = rng.integers(0, 256, size=(n, elem), dtype=np.uint8)
        x = raw.reshape(shape + (elem,))
        want = np.ascontiguousarray(np.transpose(x, axes + (rank,))).reshape(-1)
        dims, sigma = oracle.from_numpy_axes(shape, axes)
        got = oracle.naive_permute_c(raw.reshape(-1), dims, sigma, elem_bytes=elem)
        assert np.array_equal(got, want)


def test_c_oracle_rejects_bad_maps():
    with pytest.raises(ValueError):
        oracle.naive_permute_c(np.zeros(6, np.uint32), (3, 2), (0, 0))
    with pytest.raises(ValueError):
        oracle.naive_permute_c(np.zeros(5, np.uint32), (3, 2), (1, 0))


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2", "cfg3"])
def test_seeded_inputs_match_golden_digest(cfg):
    """The workload generator reproduces the bytes the golden digests were made from."""
    from paper_2506_03686_b200.workloads import CONFIGS, make_input

    ref = golden()["full_configs"][cfg]
    x = make_input(CONFIGS[cfg])
    assert sha256(x) == ref["input_sha256"]


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2", "cfg3"])
def test_c_oracle_full_config_digest(cfg):
    """C oracle at BASELINE sizes reproduces the reference's output digest."""
    from paper_2506_03686_b200.workloads import CONFIGS, make_input

    wl = CONFIGS[cfg]
    x = make_input(wl)
    dims, sigma = oracle.from_numpy_axes(wl.shape, wl.axes)
    out = oracle.naive_permute_c(x.reshape(-1).view(np.uint32), dims, sigma)
    assert sha256(out) == golden()["full_configs"][cfg]["output_sha256"]


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2", "cfg3"])
def test_reference_cpu_kernels_match_oracle(cfg):
    """The reference's emitted CPU kernels (oracle/_ref, the CPU-baseline
    arm) agree with the oracle -- emit.py's verify_native contract."""
    from oracle import refkernels
    from paper_2506_03686_b200.workloads import CONFIGS, make_input

    if not refkernels.available(cfg):
        pytest.skip("oracle/_ref not built (python oracle/build_ref.py)")
    wl = CONFIGS[cfg]
    x = make_input(wl)
    got = refkernels.RefKernel(cfg)(x)
    assert sha256(got) == golden()["full_configs"][cfg]["output_sha256"]
