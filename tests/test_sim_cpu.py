"""Host replay of the tile kernel's walk (tests/sim_tile.py) on many plans:
every shared-memory / global access in bounds and aligned, every destination
element written exactly once with the oracle's value.  No GPU needed."""

from __future__ import annotations

import numpy as np
import pytest

import oracle
import paper_2506_03686_b200 as vp
from tests.sim_tile import simulate


def _run(shape, axes, E, rng, **kw):
    prog = vp.build_program(vp.TensorLayout.from_shape(shape, E), vp.from_numpy_convention(axes), force="tile", **kw)
    n = prog.num_elements
    words = rng.integers(0, 2**63, size=n, dtype=np.uint64)
    words = words.view(np.uint32)[:n].copy() if E == 4 else words
    dims, sigma = oracle.from_numpy_axes(shape, axes)
    got = simulate(prog, words)
    assert np.array_equal(got, oracle.naive_permute_c(words, dims, sigma)), (shape, axes, prog.text)
    return prog


@pytest.mark.parametrize("E", [4, 8])
def test_sim_random_shapes(E):
    rng = np.random.default_rng(E)
    modes = {"shift": 0, "vec": 0}
    for _ in range(40):
        rank = int(rng.integers(2, 6))
        while True:
            shape = tuple(int(rng.integers(1, 24)) for _ in range(rank))
            if 64 <= np.prod(shape) <= 30000:
                break
        axes = tuple(int(a) for a in rng.permutation(rank))
        p = _run(shape, axes, E, rng)
        modes["shift"] += "aligned supersets" in p.text
        modes["vec"] += "vector elems: R 1," not in p.text
    assert modes["shift"] > 0 and modes["vec"] > 0, modes


@pytest.mark.parametrize("shape,axes", [
    ((8, 24, 20, 12), (0, 2, 3, 1)), ((64, 48), (1, 0)), ((7, 9, 13, 5, 11), (4, 1, 0, 3, 2)),
    ((17, 9, 13, 15, 3, 5), (5, 2, 0, 4, 1, 3)), ((2,) * 12, (3, 9, 0, 7, 1, 5, 2, 11, 8, 6, 4, 10)),
    ((33, 45, 19), (2, 0, 1)), ((101, 67), (1, 0)), ((6, 5, 7, 3), (1, 0, 2, 3)),
])
@pytest.mark.parametrize("E", [4, 8])
def test_sim_known_shapes(shape, axes, E):
    _run(shape, axes, E, np.random.default_rng(1))


def test_sim_campaign_sample():
    from tests.golden.pattern import golden_pattern
    from tests.helpers import golden, sha256

    cases = [c for c in golden()["cases"] if c["family"].startswith("campaign_") and 16 <= c["n"] <= 6000]
    for c in cases[:80]:
        prog = vp.build_program(vp.TensorLayout(tuple(c["dims"]), c["elem"]), vp.PermutationMap(tuple(c["sigma"])),
                                force="tile")
        out = simulate(prog, golden_pattern(c["n"], c["elem"]))
        assert sha256(out) == c["sha256"], c["name"]


def test_sim_bulk_mode(monkeypatch):
    monkeypatch.setenv("VPG_BULK", "1")
    vp.program_cache_clear()
    rng = np.random.default_rng(3)
    seen = 0
    for shape, axes, E in [((256, 96), (1, 0), 4), ((100, 76), (1, 0), 4), ((8, 24, 20, 12), (0, 2, 3, 1), 4),
                           ((2,) * 12, (3, 9, 0, 7, 1, 5, 2, 11, 8, 6, 4, 10), 8), ((36, 10, 52), (2, 0, 1), 8)]:
        p = _run(shape, axes, E, rng)
        seen += "TMA bulk" in p.text
    vp.program_cache_clear()
    assert seen >= 3
