"""Host replay of the tile kernel's walk (tests/sim_tile.py) on many plans:
every shared-memory / global access in bounds and aligned, every destination
element written exactly once with the oracle's value.  No GPU needed."""

from __future__ import annotations

import numpy as np
import pytest

import oracle
import paper_2506_03686_b200 as vp
from tests.sim_tile import simulate, simulate_exchange, tile_params


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


@pytest.mark.parametrize("E", [4, 8])
def test_sim_lin_forced(E, monkeypatch):
    """W as destination-linear 16-byte chunks (VPG_LIN=1: wherever it
    applies) on random shapes, ragged tiles and misaligned runs included."""
    monkeypatch.setenv("VPG_LIN", "1")
    vp.program_cache_clear()
    rng = np.random.default_rng(100 + E)
    lin = ragged = 0
    try:
        for _ in range(40):
            rank = int(rng.integers(2, 6))
            while True:
                shape = tuple(int(rng.integers(1, 24)) for _ in range(rank))
                if 64 <= np.prod(shape) <= 30000:
                    break
            axes = tuple(int(a) for a in rng.permutation(rank))
            p = _run(shape, axes, E, rng)
            if "W lin" in p.text:
                lin += 1
                tp = tile_params(p)
                ragged += tp.grid_a >= 0 or tp.grid_c >= 0
        for shape, axes in [((17, 9, 13, 15, 11, 27), (5, 2, 0, 4, 1, 3)), ((7, 9, 13, 5, 11), (4, 1, 0, 3, 2)),
                            ((101, 67), (1, 0)), ((33, 45, 19), (2, 0, 1))]:
            if np.prod(shape) > 200000:
                shape = shape[:-1] + (3,)
            p = _run(shape, axes, E, rng)
            lin += "W lin" in p.text
    finally:
        vp.program_cache_clear()
    assert lin >= 10 and ragged > 0, (lin, ragged)


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
    # misaligned runs: aligned supersets by bulk copy into 16-byte residue rows
    mis = 0
    for shape, axes, E in [((17, 9, 13, 15, 11, 27), (5, 2, 0, 4, 1, 3), 4), ((33, 45, 19), (2, 0, 1), 4),
                           ((101, 67), (1, 0), 4), ((7, 9, 13, 5, 11), (4, 1, 0, 3, 2), 8),
                           ((5, 3, 37, 41), (3, 0, 2, 1), 4), ((27, 31), (1, 0), 8)]:
        p = _run(shape, axes, E, rng)
        t = tile_params(p)
        mis += t.bulk == 1 and t.ph[0].rshift == 2
    vp.program_cache_clear()
    assert seen >= 3 and mis >= 3, (seen, mis)


# ------------------------------------------------------------ fused sharded exchange
EXCHANGE_CASES = [
    ((8, 6, 16, 4), (2, 0, 3, 1)),
    ((16, 12, 16, 8), (3, 1, 0, 2)),
    ((4, 64, 128), (2, 1, 0)),
    ((8, 40, 32), (0, 2, 1)),
    ((16, 6, 10, 8), (3, 2, 1, 0)),
    ((8, 8, 24, 10), (1, 3, 0, 2)),
    ((32, 5, 7, 16), (3, 1, 2, 0)),
    ((8, 3, 64, 64), (2, 3, 1, 0)),
    ((12, 2, 12, 8, 6, 6), (5, 0, 1, 3, 2, 4)),
    ((2, 2, 2, 2, 2), (2, 0, 3, 4, 1)),
    ((8, 6, 8), (0, 1, 2)),
    ((2, 16, 6, 16, 4, 8), (3, 2, 0, 1, 4, 5)),
    ((12, 12, 4), (1, 2, 0)),
    ((12, 2, 4, 16), (3, 2, 1, 0)),
    ((2,) * 12, (11, 4, 10, 1, 2, 7, 6, 0, 3, 9, 8, 5)),   # innermost source dim indexes the output shard
]


@pytest.mark.parametrize("mode", ["push", "pull"])
@pytest.mark.parametrize("G", [1, 2, 4, 8])
@pytest.mark.parametrize("E", [4, 8])
def test_sim_fused_exchange(G, E, mode):
    """push: every rank's exchange kernel reads only its input shard; pull:
    every rank's kernel writes only its output shard, reading 16-byte chunks
    that never straddle two input shards.  Together they write each output
    element exactly once with the permuted value."""
    from paper_2506_03686_b200.sharded import _programs
    from tests.golden.pattern import golden_pattern

    done = 0
    for shape, axes in EXCHANGE_CASES:
        try:
            progs = _programs(shape, axes, E, G, range(G), pull=mode == "pull")
        except vp.LayoutError:
            continue
        n = int(np.prod(shape))
        words = golden_pattern(n, E)
        got = simulate_exchange(progs, words)
        want = np.ascontiguousarray(np.transpose(words.reshape(shape), axes)).reshape(-1)
        assert np.array_equal(got, want), (shape, axes, G)
        for r, p in enumerate(progs):
            m = p.metadata
            assert m["shards"] == G and m["shard_index"] == r
        done += 1
    assert done >= (len(EXCHANGE_CASES) - 1 if G == 1 else 3)


def test_sim_negative_controls():
    """The checker is not vacuous (the reference's corrupted-table control,
    test_emit.py:156-171): corrupting one stride or extent of a valid
    parameter block is caught as an out-of-bounds access, a double write or
    a wrong value."""
    from tests.sim_tile import SimError, tile_params

    shape, axes, E = (36, 40, 44), (2, 0, 1), 4
    prog = vp.build_program(vp.TensorLayout.from_shape(shape, E), vp.from_numpy_convention(axes), force="tile")
    n = prog.num_elements
    words = np.arange(1, n + 1, dtype=np.uint32)
    dims, sigma = oracle.from_numpy_axes(shape, axes)
    want = oracle.naive_permute_c(words, dims, sigma)
    assert np.array_equal(simulate(prog, words), want)
    corruptions = []
    tp = tile_params(prog)
    for i in range(tp.ngrid):
        corruptions.append(("grid dst_stride", lambda t, i=i: setattr(t.grid[i], "dst_stride", t.grid[i].dst_stride + 1)))
        corruptions.append(("grid src_stride", lambda t, i=i: setattr(t.grid[i], "src_stride", t.grid[i].src_stride + 1)))
    corruptions.append(("W inner stride", lambda t: setattr(t.ph[1], "g_in", t.ph[1].g_in + 1)))
    corruptions.append(("R inner smem stride", lambda t: setattr(t.ph[0], "s_in", t.ph[0].s_in + 1)))
    corruptions.append(("tile count", lambda t: setattr(t, "num_tiles", t.num_tiles - 1)))
    assert len(corruptions) >= 5
    for what, fn in corruptions:
        bad = tile_params(prog)
        fn(bad)
        try:
            got = simulate(prog, words, tp=bad)
        except SimError:
            continue
        assert not np.array_equal(got, want), f"corruption of {what} went unnoticed"


def test_sim_swizzled_shifted_rows(monkeypatch):
    """Plans with the shifted-run chunk swizzle (misaligned runs, opt-in
    VPG_SWZ=1) replay bit-exact: R writes and W reads agree on the layout."""
    monkeypatch.setenv("VPG_SWZ", "1")
    monkeypatch.setenv("VPG_NO_RES", "1")      # residue row strides would win the cost model
    vp.program_cache_clear()
    rng = np.random.default_rng(11)
    n_swz = 0
    for _ in range(120):
        r = int(rng.integers(2, 6))
        shape = tuple(int(x) for x in rng.integers(2, 30, size=r))
        axes = tuple(int(a) for a in rng.permutation(r))
        E = int(rng.choice([4, 8]))
        prog = vp.build_program(vp.TensorLayout.from_shape(shape, E), vp.from_numpy_convention(axes), force="tile")
        if "swizzle" not in prog.text:
            continue
        n = prog.num_elements
        words = rng.integers(0, 2**63, size=n, dtype=np.uint64)
        words = words.view(np.uint32)[:n].copy() if E == 4 else words
        dims, sigma = oracle.from_numpy_axes(shape, axes)
        assert np.array_equal(simulate(prog, words), oracle.naive_permute_c(words, dims, sigma)), (shape, axes, E)
        n_swz += 1
        if n_swz >= 25:
            break
    vp.program_cache_clear()
    assert n_swz >= 10


def test_sim_residue_rows():
    """Misaligned runs with residue row strides (the default shifted-run
    layout): R lands every 16-byte aligned source chunk on an aligned smem
    chunk and W reads affine offsets; replays bit-exact against the C
    oracle, including ragged tiles and 8-byte words."""
    vp.program_cache_clear()
    rng = np.random.default_rng(23)
    n_res = 0
    for _ in range(300):
        r = int(rng.integers(2, 6))
        shape = tuple(int(x) for x in rng.integers(2, 40, size=r))
        axes = tuple(int(a) for a in rng.permutation(r))
        E = int(rng.choice([4, 8]))
        prog = vp.build_program(vp.TensorLayout.from_shape(shape, E), vp.from_numpy_convention(axes), force="tile")
        if tile_params(prog).rres == 0:
            continue
        n = prog.num_elements
        words = rng.integers(0, 2**63, size=n, dtype=np.uint64)
        words = words.view(np.uint32)[:n].copy() if E == 4 else words
        dims, sigma = oracle.from_numpy_axes(shape, axes)
        assert np.array_equal(simulate(prog, words), oracle.naive_permute_c(words, dims, sigma)), (shape, axes, E)
        n_res += 1
        if n_res >= 40:
            break
    assert n_res >= 20


def test_sim_w2_blocks():
    """W in V x V register-transposed blocks on the congruent swizzled
    layout (16-byte smem loads and 16-byte destination stores): bit-exact
    replay on shapes where the planner picks it, 4- and 8-byte words, ragged
    tiles included."""
    vp.program_cache_clear()
    rng = np.random.default_rng(31)
    n_w2 = 0
    shapes = [((64, 256), (1, 0)), ((96, 128), (1, 0)), ((8, 64, 40), (0, 2, 1)), ((3, 32, 64, 8), (1, 3, 2, 0))]
    for _ in range(400):
        r = int(rng.integers(2, 5))
        shapes.append((tuple(int(x) for x in rng.choice([4, 8, 12, 16, 32, 64, 128], size=r)),
                       tuple(int(a) for a in rng.permutation(r))))
    for shape, axes in shapes:
        if np.prod(shape) > 300000:
            continue
        for E in (4, 8):
            prog = vp.build_program(vp.TensorLayout.from_shape(shape, E), vp.from_numpy_convention(axes), force="tile")
            if tile_params(prog).ph[1].w2 == 0:
                continue
            n = prog.num_elements
            words = rng.integers(0, 2**63, size=n, dtype=np.uint64)
            words = words.view(np.uint32)[:n].copy() if E == 4 else words
            dims, sigma = oracle.from_numpy_axes(shape, axes)
            assert np.array_equal(simulate(prog, words), oracle.naive_permute_c(words, dims, sigma)), (shape, axes, E)
            n_w2 += 1
        if n_w2 >= 25:
            break
    assert n_w2 >= 10, n_w2


def test_sim_golden_cases_with_swizzled_layouts():
    """Every reference golden case (up to 70k elements) whose plan uses the
    congruent swizzled layout or V x V blocks replays to the reference's
    recorded digest."""
    from tests.golden.pattern import golden_pattern
    from tests.helpers import golden, sha256

    ran = 0
    for c in golden()["cases"]:
        if c["n"] > 70000:
            continue
        prog = vp.build_program(vp.TensorLayout(tuple(c["dims"]), c["elem"]), vp.PermutationMap(tuple(c["sigma"])))
        if prog.kernel != "tile":
            continue
        t = tile_params(prog)
        if not (t.ph[1].w2 or t.ph[0].swz):
            continue
        assert sha256(simulate(prog, golden_pattern(c["n"], c["elem"]))) == c["sha256"], c["name"]
        ran += 1
    assert ran >= 10


def test_sim_narrow_gather_blocks():
    """W in narrow gather blocks (1- and 2-byte words whose
    destination-innermost extent is a multiple of 2, 4 or 8 but not of V):
    g scalar smem loads packed into one 4- or 8-byte store; bit-exact replay
    with misaligned source runs (residue rows) and ragged tiles."""
    vp.program_cache_clear()
    rng = np.random.default_rng(77)
    seen = {}
    shapes = [((20, 516, 999), (0, 2, 1)), ((3, 36, 211), (0, 2, 1)), ((5, 12, 203), (2, 1, 0)),
              ((6, 44, 10, 67), (0, 3, 2, 1)), ((4, 18, 301), (0, 2, 1)), ((2, 250, 333), (0, 2, 1))]
    for _ in range(300):
        r = int(rng.integers(2, 5))
        dims = [int(rng.choice([2, 3, 4, 6, 10, 12, 20, 28, 36, 44, 52, 100, 204])) for _ in range(r - 1)]
        dims.append(int(rng.choice([33, 67, 99, 131, 203, 301])))
        shapes.append((tuple(dims), tuple(int(a) for a in rng.permutation(r))))
    for shape, axes in shapes:
        if np.prod(shape) > 400000:
            continue
        for E in (1, 2):
            prog = vp.build_program(vp.TensorLayout.from_shape(shape, E), vp.from_numpy_convention(axes), force="tile")
            w2 = tile_params(prog).ph[1].w2
            if w2 <= 64:
                continue
            assert "gather blocks of" in prog.text
            n = prog.num_elements
            words = rng.integers(0, 256 ** E, size=n, dtype=np.uint64).astype({1: np.uint8, 2: np.uint16}[E])
            dims, sigma = oracle.from_numpy_axes(shape, axes)
            assert np.array_equal(simulate(prog, words), oracle.naive_permute_c(words, dims, sigma)), (shape, axes, E)
            seen[(E, w2 - 64)] = seen.get((E, w2 - 64), 0) + 1
        if sum(seen.values()) >= 24 and len(seen) >= 3:
            break
    assert len(seen) >= 3 and sum(seen.values()) >= 10, seen


def test_sim_narrow_w_vectors():
    """Narrow W vectors on residue rows (1- and 2-byte words, source runs
    misaligned to 16 bytes but aligned to 4 or 8): one 4- or 8-byte smem load
    per 2-8 elements of source dim 0, stored element by element; bit-exact
    replay with the smem vector alignment checked."""
    vp.program_cache_clear()
    rng = np.random.default_rng(3)
    seen = {}
    shapes = [((300, 1012), (1, 0)), ((37, 20, 500), (2, 0, 1)), ((33, 100, 77), (1, 2, 0)), ((45, 36, 210), (2, 1, 0)),
              ((129, 1004), (1, 0)), ((7, 9, 36, 52), (3, 1, 0, 2)), ((77, 1000), (1, 0)), ((31, 40, 99), (2, 0, 1))]
    for _ in range(300):
        r = int(rng.integers(2, 5))
        dims = [int(rng.choice([3, 5, 7, 9, 33, 67, 101])) for _ in range(r - 1)]
        dims.append(int(rng.choice([20, 24, 36, 40, 44, 52, 100, 204, 1012, 18, 42, 90, 250])))
        shapes.append((tuple(dims), tuple(int(a) for a in rng.permutation(r))))
    for shape, axes in shapes:
        if np.prod(shape) > 400000 or np.prod(shape) < 2000:
            continue
        for E in (1, 2):
            prog = vp.build_program(vp.TensorLayout.from_shape(shape, E), vp.from_numpy_convention(axes), force="tile")
            v = tile_params(prog).ph[1].vec
            if v <= 1 or v * E >= 16:
                continue
            assert "residue row strides" in prog.text
            n = prog.num_elements
            words = rng.integers(0, 256 ** E, size=n, dtype=np.uint64).astype({1: np.uint8, 2: np.uint16}[E])
            dims, sigma = oracle.from_numpy_axes(shape, axes)
            assert np.array_equal(simulate(prog, words), oracle.naive_permute_c(words, dims, sigma)), (shape, axes, E)
            seen[(E, v)] = seen.get((E, v), 0) + 1
        if sum(seen.values()) >= 30 and len(seen) >= 3:
            break
    assert len(seen) >= 3 and sum(seen.values()) >= 12, seen
