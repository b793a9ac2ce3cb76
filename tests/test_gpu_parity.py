"""GPU parity: the CUDA path against the reference's own golden vectors and
the CPU oracle, bit-exact (pure data movement: any byte difference is a bug).

Golden vectors come from the reference itself (tests/golden/make_golden.py);
the C oracle (oracle/naive_permute.c) is pinned against the same vectors in
tests/test_oracle.py.
"""

from __future__ import annotations

import numpy as np
import pytest

from tests.golden.pattern import golden_pattern
from tests.helpers import golden, gpu_permute_bytes, sha256

pytestmark = pytest.mark.gpu


def _cases(families=None):
    return [c for c in golden()["cases"] if families is None or c["family"] in families]


@pytest.mark.parametrize("force", [None, "tile", "gather"])
def test_golden_small_cases(cuda, force):
    """Known answers, paper shape, Appendix-A edges, merge cases, ragged sweep
    (test_core.py:93-100,147-151; test_cli.py:69-83; test_acceptance.py:239-274)."""
    cases = _cases({"known", "paper", "merge", "edge", "ragged"})
    assert len(cases) > 100
    for c in cases:
        data = golden_pattern(c["n"], c["elem"])
        out, prog = gpu_permute_bytes(c["dims"], c["sigma"], c["elem"], data, force=force)
        assert sha256(out) == c["sha256"], (c["name"], prog.text)
        if "out" in c:
            words = out.view(np.uint32 if c["elem"] == 4 else np.uint64)
            assert words.tolist() == c["out"], c["name"]


def test_known_answer_2x3(cuda):
    """test_core.py:147-151: (2,3) transpose of arange -> [0,3,1,4,2,5]."""
    data = np.arange(6, dtype=np.uint32)
    for force in (None, "tile", "gather"):
        out, _ = gpu_permute_bytes((3, 2), (1, 0), 4, data, force=force)
        assert out.view(np.uint32).tolist() == [0, 3, 1, 4, 2, 5]


def test_bit_reversal_2x2x2(cuda):
    """test_core.py:93-100: full role reversal on (2,2,2) is bit reversal."""
    data = np.arange(8, dtype=np.uint32)
    for force in (None, "tile", "gather"):
        out, _ = gpu_permute_bytes((2, 2, 2), (2, 1, 0), 4, data, force=force)
        assert out.view(np.uint32).tolist() == [0, 4, 2, 6, 1, 5, 3, 7]


@pytest.mark.parametrize("force", [None, "tile"])
def test_reference_campaign_1000(cuda, force):
    """The reference's 1000-case randomized campaign (seed 2024, ranks 2-16,
    <= 2^16 elements; test_acceptance.py:25-33), bitwise on the GPU."""
    cases = [c for c in golden()["cases"] if c["family"].startswith("campaign_")]
    assert len(cases) == 1000
    fams = {}
    bad = []
    for c in cases:
        data = golden_pattern(c["n"], c["elem"])
        out, prog = gpu_permute_bytes(c["dims"], c["sigma"], c["elem"], data, force=force)
        fams[c["family"]] = fams.get(c["family"], 0) + 1
        if sha256(out) != c["sha256"]:
            bad.append((c["name"], c["shape"], c["axes"], prog.kernel))
    assert not bad, bad[:5]
    assert all(v > 0 for v in fams.values()) and len(fams) == 3


def test_full_size_2pow20(cuda):
    """N = 2^20 transpose (test_acceptance.py:35-44)."""
    c = next(c for c in golden()["cases"] if c["name"] == "full_1024x1024")
    out, _ = gpu_permute_bytes(c["dims"], c["sigma"], 4, golden_pattern(c["n"], 4))
    assert sha256(out) == c["sha256"]


@pytest.mark.parametrize("elem", [1, 2, 16])
def test_extra_elem_widths_vs_oracle(cuda, elem):
    """Superset element widths (the reference accepts 4/8 only, core.py:29)
    against the C oracle, which is pinned on 4/8 by the golden vectors."""
    import oracle

    rng = np.random.default_rng(100 + elem)
    for t in range(40):
        rank = int(rng.integers(1, 6))
        dims = tuple(int(rng.integers(1, 12)) for _ in range(rank))
        sigma = tuple(int(x) for x in rng.permutation(rank))
        n = int(np.prod(dims))
        data = rng.integers(0, 256, size=n * elem, dtype=np.uint8)
        want = oracle.naive_permute_c(data.view(np.uint8), dims, sigma, elem_bytes=elem)
        for force in (None, "tile", "gather"):
            out, prog = gpu_permute_bytes(dims, sigma, elem, data, force=force)
            assert np.array_equal(out, want.view(np.uint8)), (dims, sigma, force, prog.text)


def test_random_general_vs_oracle_large(cuda):
    """Larger random shapes (odd dims, up to ~4M elements) against the C
    oracle, 64-bit random words (high halves set)."""
    import oracle

    rng = np.random.default_rng(7)
    for t in range(60):
        rank = int(rng.integers(2, 7))
        while True:
            dims = tuple(int(rng.integers(1, 40)) for _ in range(rank))
            if np.prod(dims) <= (1 << 22):
                break
        sigma = tuple(int(x) for x in rng.permutation(rank))
        elem = int(rng.choice([4, 8]))
        n = int(np.prod(dims))
        data = rng.integers(0, 2**63, size=n, dtype=np.uint64)
        data = data.view(np.uint32)[:n].copy() if elem == 4 else data
        want = oracle.naive_permute_c(data, dims, sigma)
        out, prog = gpu_permute_bytes(dims, sigma, elem, data)
        assert np.array_equal(out, want.view(np.uint8)), (dims, sigma, elem, prog.text)


def test_golden_cases_specialised_kernels(cuda):
    """Per-case NVRTC-specialised tile kernels (jit.cpp) on the known-answer,
    paper, merge, edge and ragged cases plus a seeded sample of the
    reference campaign."""
    import random

    cases = _cases({"known", "paper", "merge", "edge"})
    camp = [c for c in golden()["cases"] if c["family"].startswith("campaign_") and c["n"] > 1]
    random.Random(7).shuffle(camp)
    cases += camp[:60] + _cases({"ragged"})[:20]
    for c in cases:
        data = golden_pattern(c["n"], c["elem"])
        from paper_2506_03686_b200 import PermutationMap, TensorLayout, build_program
        from paper_2506_03686_b200.api import execute_device
        import torch

        prog = build_program(TensorLayout(tuple(c["dims"]), c["elem"]), PermutationMap(tuple(c["sigma"])),
                             force="tile", jit=True)
        x = torch.from_numpy(data.view(np.uint8).copy()).cuda()
        out = execute_device(prog, x).cpu().numpy().reshape(-1)
        assert prog.jit_state == 2, (c["name"], "specialised kernel not loaded")
        assert sha256(out) == c["sha256"], (c["name"], prog.text)


@pytest.mark.parametrize("elem", [4, 8])
@pytest.mark.parametrize("jit", [False, True])
def test_shifted_run_reads_misaligned_dims(cuda, elem, jit):
    """Odd dims make every source run start off 16-byte alignment; the tile
    reads 16-byte aligned supersets and shifts in smem (planner: 'aligned
    supersets').  Checked against the C oracle, including the buffer's last
    run (bounds-clipped final chunk) and ragged tiles."""
    import oracle
    from paper_2506_03686_b200 import PermutationMap, TensorLayout, build_program

    rng = np.random.default_rng(elem + 10 * jit)
    shapes = [((7, 9, 13, 5, 11, 27), (5, 2, 0, 4, 1, 3)), ((17, 9, 13, 15, 11, 27), (5, 2, 0, 4, 1, 3)),
              ((33, 45, 19), (2, 0, 1)), ((5, 7, 9, 11, 13), (4, 3, 2, 1, 0)), ((101, 67), (1, 0)),
              ((3, 77, 5, 31), (1, 3, 0, 2))]
    seen_shift = 0
    for shape, axes in shapes:
        dims, sigma = oracle.from_numpy_axes(shape, axes)
        n = int(np.prod(shape))
        data = rng.integers(0, 2**63, size=n, dtype=np.uint64)
        data = data.view(np.uint32)[:n].copy() if elem == 4 else data
        prog = build_program(TensorLayout(dims, elem), PermutationMap(sigma), force="tile", jit=jit)
        seen_shift += "aligned supersets" in prog.text
        out, _ = gpu_permute_bytes(dims, sigma, elem, data, force="tile", jit=jit)
        want = oracle.naive_permute_c(data, dims, sigma)
        assert np.array_equal(out, want.view(np.uint8)), (shape, axes, prog.text)
    assert seen_shift >= 2


@pytest.mark.parametrize("jit,count", [(False, 120), (True, 20)])
def test_large_random_campaign(cuda, jit, count):
    """Beyond the reference's <= 2^16-element campaign: 2^16..2^21-element
    random shapes (odd, pow2 and all-2 families, 4/8-byte words), checked
    against torch's own device permute and the inverse round trip."""
    import torch

    from paper_2506_03686_b200 import TensorLayout, build_program, from_numpy_convention, permuted_layout
    from paper_2506_03686_b200.api import execute_device

    rng = np.random.default_rng(31 + jit)
    for i in range(count):
        fam = i % 3
        while True:
            rank = int(rng.integers(2, 9))
            if fam == 0:
                shape = tuple(int(rng.integers(2, 40)) for _ in range(rank))
            elif fam == 1:
                shape = tuple(int(2 ** rng.integers(1, 7)) for _ in range(rank))
            else:
                shape = (2,) * int(rng.integers(16, 22))
            n = int(np.prod(shape))
            if (1 << 16) <= n <= (1 << 21):
                break
        axes = tuple(int(a) for a in rng.permutation(len(shape)))
        elem = int(rng.choice([4, 8]))
        word = torch.int32 if elem == 4 else torch.int64
        x = torch.randint(-2**31, 2**31 - 1, shape, dtype=word, device=cuda)
        prog = build_program(TensorLayout.from_shape(shape, elem), from_numpy_convention(axes), jit=jit)
        y = execute_device(prog, x)
        if len(shape) <= 25:
            assert torch.equal(y, x.permute(axes).contiguous()), (shape, axes, prog.text)
        inv = build_program(permuted_layout(prog.layout, prog.pmap), prog.pmap.inverse(), jit=jit)
        assert torch.equal(execute_device(inv, y).reshape(-1), x.reshape(-1)), (shape, axes)
        if jit and prog.kernel == "tile":
            assert prog.jit_state == 2


@pytest.mark.parametrize("jit", [False, True])
def test_bulk_tma_mode(cuda, jit, monkeypatch):
    """Opt-in R phase as TMA bulk copies (producer warp + mbarriers,
    VPG_BULK=1): bit-exact on transposes, batched transposes, all-2 ranks and
    ragged tiles."""
    import torch

    from paper_2506_03686_b200 import TensorLayout, build_program, from_numpy_convention, program_cache_clear
    from paper_2506_03686_b200.api import execute_device

    monkeypatch.setenv("VPG_BULK", "1")
    program_cache_clear()
    seen = 0
    for shape, axes, E in [((256, 384), (1, 0), 4), ((1000, 776), (1, 0), 4), ((8, 24, 20, 12), (0, 2, 3, 1), 4),
                           ((2,) * 18, tuple(np.random.default_rng(4).permutation(18).tolist()), 8),
                           ((36, 100, 52), (2, 0, 1), 8)]:
        prog = build_program(TensorLayout.from_shape(shape, E), from_numpy_convention(axes), force="tile", jit=jit)
        seen += "TMA bulk" in prog.text
        dt = torch.int32 if E == 4 else torch.int64
        x = torch.randint(-2**30, 2**30, shape, dtype=dt, device=cuda)
        assert torch.equal(execute_device(prog, x), x.permute(axes).contiguous()), (shape, prog.text)
    program_cache_clear()
    assert seen >= 3


def test_negative_controls(cuda):
    """The parity checks are not vacuous: a kernel run with a different map,
    or an output with one word changed, fails the same comparisons the
    parity tests use (digest and oracle)."""
    import oracle

    cases = [c for c in golden()["cases"] if c["family"].startswith("campaign_") and c["n"] >= 256][:20]
    assert cases
    ran = 0
    for c in cases:
        data = golden_pattern(c["n"], c["elem"])
        out, _ = gpu_permute_bytes(c["dims"], c["sigma"], c["elem"], data)
        assert sha256(out) == c["sha256"]
        flipped = out.copy()
        flipped[len(flipped) // 2] ^= 1
        assert sha256(flipped) != c["sha256"]
        # a different (rotated) map over the same dims must not reproduce the digest
        rot = tuple(c["sigma"][1:]) + (c["sigma"][0],)
        want = oracle.naive_permute_c(data, c["dims"], c["sigma"]).reshape(-1).view(np.uint8)
        other = oracle.naive_permute_c(data, c["dims"], rot).reshape(-1).view(np.uint8)
        if np.array_equal(want, other):
            continue                     # the rotated map is the same bijection here
        wrong, _ = gpu_permute_bytes(c["dims"], rot, c["elem"], data)
        assert sha256(wrong) != c["sha256"], c["name"]
        assert not np.array_equal(wrong, want)
        ran += 1
    assert ran >= 10


@pytest.mark.parametrize("jit", [False, True])
def test_swizzled_shifted_rows_opt_in(cuda, jit, monkeypatch):
    """The opt-in chunk swizzle of shifted rows (VPG_SWZ=1) stays bit-exact
    on misaligned shapes, specialised and ahead-of-time kernels."""
    import torch

    import paper_2506_03686_b200 as vp
    from paper_2506_03686_b200.api import execute_device

    monkeypatch.setenv("VPG_SWZ", "1")
    monkeypatch.setenv("VPG_NO_RES", "1")      # residue row strides would win the cost model
    vp.program_cache_clear()
    rng = np.random.default_rng(5)
    done = 0
    for _ in range(200):
        r = int(rng.integers(2, 6))
        shape = tuple(int(x) for x in rng.integers(2, 40, size=r))
        axes = tuple(int(a) for a in rng.permutation(r))
        E = int(rng.choice([4, 8]))
        prog = vp.build_program(vp.TensorLayout.from_shape(shape, E), vp.from_numpy_convention(axes),
                                force="tile", jit=jit)
        if "swizzle" not in prog.text:
            continue
        n = int(np.prod(shape))
        x = torch.randint(-2**31, 2**31 - 1, (n * E // 4,), dtype=torch.int32, device="cuda")
        xv = x.view(torch.int32 if E == 4 else torch.int64).view(shape)
        y = execute_device(prog, x.view(torch.uint8))
        assert torch.equal(y.view(xv.dtype).view(-1), xv.permute(axes).reshape(-1)), (shape, axes, E)
        done += 1
        if done >= (6 if jit else 20):
            break
    vp.program_cache_clear()
    assert done >= 5


@pytest.mark.parametrize("jit", [False, True])
def test_residue_row_strides(cuda, jit):
    """Misaligned runs with residue row strides (default layout for shifted
    runs): every tile starts at its own offset modulo 16 bytes inside the
    staging buffer; bit-exact on random shapes, 4- and 8-byte words,
    specialised and ahead-of-time kernels, ragged tiles included."""
    import torch

    import paper_2506_03686_b200 as vp
    from paper_2506_03686_b200.api import execute_device

    from tests.sim_tile import tile_params

    rng = np.random.default_rng(17)
    done = 0
    for _ in range(400):
        r = int(rng.integers(2, 7))
        shape = tuple(int(x) for x in rng.integers(2, 48, size=r))
        if np.prod(shape) > (1 << 22):
            continue
        axes = tuple(int(a) for a in rng.permutation(r))
        E = int(rng.choice([4, 8]))
        prog = vp.build_program(vp.TensorLayout.from_shape(shape, E), vp.from_numpy_convention(axes),
                                force="tile", jit=jit)
        if tile_params(prog).rres == 0:
            continue
        n = int(np.prod(shape))
        x = torch.randint(-2**31, 2**31 - 1, (n * E // 4,), dtype=torch.int32, device="cuda")
        xv = x.view(torch.int32 if E == 4 else torch.int64).view(shape)
        y = execute_device(prog, x.view(torch.uint8))
        assert torch.equal(y.view(xv.dtype).view(-1), xv.permute(axes).reshape(-1)), (shape, axes, E)
        done += 1
        if done >= (12 if jit else 40):
            break
    assert done >= 8



@pytest.mark.parametrize("jit", [False, True])
def test_w2_blocks(cuda, jit):
    """W in V x V register-transposed blocks with 16-byte stores (congruent
    swizzled layout): bit-exact on shapes where the planner picks it, 4- and
    8-byte words, specialised and ahead-of-time kernels, ragged tiles; a
    destination off 16-byte alignment takes the scalar-store variant."""
    import torch

    import paper_2506_03686_b200 as vp
    from paper_2506_03686_b200.api import execute_device
    from tests.sim_tile import tile_params

    rng = np.random.default_rng(41)
    done = 0
    shapes = [((64, 256), (1, 0)), ((4096, 4096), (1, 0)), ((32, 64, 56, 56), (0, 2, 3, 1)), ((96, 128), (1, 0))]
    for _ in range(300):
        r = int(rng.integers(2, 5))
        shapes.append((tuple(int(x) for x in rng.choice([4, 8, 12, 16, 32, 64, 128, 192], size=r)),
                       tuple(int(a) for a in rng.permutation(r))))
    for shape, axes in shapes:
        n = int(np.prod(shape))
        if n > (1 << 24):
            continue
        E = 8 if (done % 3 == 2) else 4
        prog = vp.build_program(vp.TensorLayout.from_shape(shape, E), vp.from_numpy_convention(axes),
                                force="tile", jit=jit)
        if tile_params(prog).ph[1].w2 == 0:
            continue
        x = torch.randint(-2**31, 2**31 - 1, (n * E // 4,), dtype=torch.int32, device="cuda")
        xv = x.view(torch.int32 if E == 4 else torch.int64).view(shape)
        want = xv.permute(axes).reshape(-1)
        y = execute_device(prog, x.view(torch.uint8))
        assert torch.equal(y.view(xv.dtype).view(-1), want), (shape, axes, E)
        big = torch.empty(n * E + E, dtype=torch.uint8, device="cuda")
        out = big[E:]                      # destination off 16-byte alignment by one element
        execute_device(prog, x.view(torch.uint8), out=out)
        assert torch.equal(out.view(xv.dtype), want), (shape, axes, E, "misaligned dst")
        done += 1
        if done >= (8 if jit else 24):
            break
    assert done >= 6


@pytest.mark.parametrize("jit", [True, False])
def test_lin_w_mode(cuda, jit, monkeypatch):
    """W as destination-linear 16-byte chunks (VPG_LIN=1, opt-in): bit-exact
    on misaligned and ragged shapes, 4- and 8-byte words, both kernel
    builds, a destination buffer off its 16-byte alignment (the chunk grid
    follows the address) -- cfg3's shape included."""
    import torch

    import paper_2506_03686_b200 as vp
    from paper_2506_03686_b200.api import execute_device

    monkeypatch.setenv("VPG_LIN", "1")
    vp.program_cache_clear()
    rng = np.random.default_rng(77)
    shapes = [((17, 9, 13, 15, 11, 27), (5, 2, 0, 4, 1, 3)), ((7, 9, 13, 5, 11), (4, 1, 0, 3, 2)),
              ((101, 67), (1, 0)), ((33, 45, 19), (2, 0, 1)), ((13, 7, 300), (2, 1, 0))]
    for _ in range(60):
        r = int(rng.integers(2, 6))
        shapes.append((tuple(int(x) for x in rng.integers(3, 40, size=r)), tuple(int(a) for a in rng.permutation(r))))
    done = 0
    try:
        for i, (shape, axes) in enumerate(shapes):
            n = int(np.prod(shape))
            if n > (1 << 23) or n < 4096:
                continue
            E = 8 if i % 3 == 2 else 4
            prog = vp.build_program(vp.TensorLayout.from_shape(shape, E), vp.from_numpy_convention(axes),
                                    force="tile", jit=jit)
            if "W lin" not in prog.text:
                continue
            x = torch.randint(-2**31, 2**31 - 1, (n * E // 4,), dtype=torch.int32, device="cuda")
            xv = x.view(torch.int32 if E == 4 else torch.int64).view(shape)
            want = xv.permute(axes).reshape(-1)
            y = execute_device(prog, x.view(torch.uint8))
            assert torch.equal(y.view(xv.dtype).view(-1), want), (shape, axes, E, prog.text)
            big = torch.empty(n * E + E, dtype=torch.uint8, device="cuda")
            out = big[E:]
            execute_device(prog, x.view(torch.uint8), out=out)
            assert torch.equal(out.view(xv.dtype), want), (shape, axes, E, "misaligned dst")
            done += 1
            if jit and done >= 12:
                break
    finally:
        vp.program_cache_clear()
    assert done >= 10, done


@pytest.mark.parametrize("shape,axes,elem,mode", [
    ((32, 64, 56, 56), (0, 2, 3, 1), 2, "VxV"),            # fp16 NCHW -> NHWC
    ((2048, 1024), (1, 0), 1, "VxV"),                       # byte transpose
    ((1024, 768), (1, 0), 1, "R 16"),
    ((17, 9, 13, 15, 11, 27), (5, 2, 0, 4, 1, 3), 2, "aligned supersets"),   # cfg3's shape in fp16
    ((1027, 515), (1, 0), 1, "aligned supersets"),          # odd byte transpose
    ((8, 512, 7, 7), (0, 2, 3, 1), 2, "aligned supersets"),   # 7x7 feature maps
    ((16, 64, 32, 128), (0, 2, 1, 3), 2, "R 8"),
])
def test_small_words_vectorised(cuda, shape, axes, elem, mode):
    """1- and 2-byte words (fp16/bf16, bytes) move as 16-byte vectors: V x V
    register-transposed blocks with 16-byte stores on aligned tiles, aligned
    supersets of misaligned runs into residue rows otherwise; bit-exact
    against torch, specialised and ahead-of-time kernels, a misaligned
    destination included."""
    import torch

    import paper_2506_03686_b200 as vp
    from paper_2506_03686_b200.api import execute_device

    dt = {1: torch.uint8, 2: torch.int16}[elem]
    n = int(np.prod(shape))
    for jit in (True, False):
        prog = vp.build_program(vp.TensorLayout.from_shape(shape, elem), vp.from_numpy_convention(axes),
                                force="tile", jit=jit)
        assert mode in prog.text, prog.text
        x = torch.randint(0, 255, (n * elem,), dtype=torch.uint8, device="cuda")
        want = x.view(dt).view(shape).permute(axes).reshape(-1)
        y = execute_device(prog, x)
        assert torch.equal(y.view(dt).view(-1), want), (shape, axes, elem, jit)
        big = torch.empty(n * elem + elem, dtype=torch.uint8, device="cuda")
        execute_device(prog, x, out=big[elem:])
        assert torch.equal(big[elem:].view(dt), want), (shape, axes, elem, jit, "misaligned dst")


@pytest.mark.parametrize("shape,axes,elem", [
    ((8, 3, 256, 256), (0, 2, 3, 1), 1),      # u8 image CHW -> HWC
    ((8, 3, 256, 256), (0, 2, 3, 1), 2),      # bf16
    ((8, 3, 256, 256), (0, 2, 3, 1), 4),      # f32
    ((4, 4, 128, 384), (0, 2, 3, 1), 1),      # RGBA
    ((64, 2, 4096), (0, 2, 1), 4),            # (re, im) planes -> interleaved
    ((16, 5, 96, 64), (0, 2, 3, 1), 2),       # k = 5
])
def test_interleave_blocks(cuda, shape, axes, elem):
    """W in k x V interleave blocks (a small destination-innermost dim, k =
    2..8, after source dim 0): k 16-byte smem vectors -> k 16-byte stores;
    bit-exact against torch, specialised and ahead-of-time kernels."""
    import torch

    import paper_2506_03686_b200 as vp
    from paper_2506_03686_b200.api import execute_device

    dt = {1: torch.uint8, 2: torch.int16, 4: torch.int32}[elem]
    n = int(np.prod(shape))
    seen = 0
    for jit in (True, False):
        prog = vp.build_program(vp.TensorLayout.from_shape(shape, elem), vp.from_numpy_convention(axes),
                                force="tile", jit=jit)
        seen += "interleave" in prog.text
        x = torch.randint(0, 255, (n * elem,), dtype=torch.uint8, device="cuda")
        want = x.view(dt).view(shape).permute(axes).reshape(-1)
        y = execute_device(prog, x)
        assert torch.equal(y.view(dt).view(-1), want), (shape, axes, elem, jit)
    assert seen >= 1, prog.text


@pytest.mark.parametrize("shape,axes,elem", [
    ((8, 512, 16, 64), (0, 2, 1, 3), 2),     # attention head split, bf16, 128-byte rows
    ((8, 512, 16, 64), (0, 2, 1, 3), 1),     # u8, 64-byte rows
    ((4, 256, 12, 32), (0, 2, 1, 3), 4),     # f32, 128-byte rows
    ((3, 5, 7, 96), (2, 0, 1, 3), 2),
])
def test_short_rows_vector_stores(cuda, shape, axes, elem):
    """Stride-1-preserving permutations with rows below the rows kernel's
    512 bytes run on the tile kernel with each 16-byte smem vector stored as
    one 16-byte destination chunk; bit-exact, aligned and misaligned
    destinations (the latter takes the scalar-store variant)."""
    import torch

    import paper_2506_03686_b200 as vp
    from paper_2506_03686_b200.api import execute_device

    dt = {1: torch.uint8, 2: torch.int16, 4: torch.int32}[elem]
    n = int(np.prod(shape))
    for jit in (True, False):
        prog = vp.build_program(vp.TensorLayout.from_shape(shape, elem), vp.from_numpy_convention(axes), jit=jit)
        assert prog.kernel == "tile"
        x = torch.randint(0, 255, (n * elem,), dtype=torch.uint8, device="cuda")
        want = x.view(dt).view(shape).permute(axes).reshape(-1)
        assert torch.equal(execute_device(prog, x).view(dt).view(-1), want), (shape, jit)
        big = torch.empty(n * elem + elem, dtype=torch.uint8, device="cuda")
        execute_device(prog, x, out=big[elem:])
        assert torch.equal(big[elem:].view(dt), want), (shape, jit, "misaligned dst")


@pytest.mark.parametrize("shape,axes,elem", [
    ((16, 256, 1000), (0, 2, 1), 1),          # u8 batched transpose, misaligned source runs
    ((4, 512, 999), (0, 2, 1), 2),
    ((80, 17, 59), (1, 2, 0), 1),
    ((16, 18, 38), (2, 1, 0), 4),
    ((10, 10, 47, 17), (0, 3, 2, 1), 8),
    ((20, 516, 999), (0, 2, 1), 1),           # narrow blocks: 4 u8 -> one 4-byte store
    ((26, 26, 333), (1, 2, 0), 2),            # 2 u16 -> one 4-byte store
    ((6, 44, 10, 67), (0, 3, 2, 1), 1),
    ((3, 36, 2111), (0, 2, 1), 2),            # 4 u16 -> one 8-byte store
])
def test_gather_blocks(cuda, shape, axes, elem):
    """W in gather blocks: V destination-innermost elements from V smem rows
    (residue rows included) packed into one 16-byte store; bit-exact,
    specialised and ahead-of-time kernels, a misaligned destination (scalar
    variant) included."""
    import torch

    import paper_2506_03686_b200 as vp
    from paper_2506_03686_b200.api import execute_device

    dt = {1: torch.uint8, 2: torch.int16, 4: torch.int32, 8: torch.int64}[elem]
    n = int(np.prod(shape))
    seen = 0
    for jit in (True, False):
        prog = vp.build_program(vp.TensorLayout.from_shape(shape, elem), vp.from_numpy_convention(axes),
                                force="tile", jit=jit)
        seen += "gather blocks" in prog.text
        x = torch.randint(0, 255, (n * elem,), dtype=torch.uint8, device="cuda")
        want = x.view(dt).view(shape).permute(axes).reshape(-1)
        assert torch.equal(execute_device(prog, x).view(dt).view(-1), want), (shape, jit)
        big = torch.empty(n * elem + elem, dtype=torch.uint8, device="cuda")
        execute_device(prog, x, out=big[elem:])
        assert torch.equal(big[elem:].view(dt), want), (shape, jit, "misaligned dst")
    assert seen >= 1, prog.text


@pytest.mark.parametrize("shape,axes,elem", [
    ((3000, 1012), (1, 0), 1),                # 4-byte W vectors of u8
    ((1290, 1004), (1, 0), 2),                # 4-byte W vectors of u16 (2 elements)
    ((45, 36, 2100), (2, 1, 0), 1),
    ((777, 67, 56), (2, 1, 0), 1),            # 8-byte W vectors of u8
    ((301, 67, 100), (2, 0, 1), 2),           # 8-byte W vectors of u16
])
def test_narrow_w_vectors(cuda, shape, axes, elem):
    """Narrow W vectors on residue rows: bit-exact, specialised and
    ahead-of-time kernels, a source buffer misaligned to 16 bytes (scalar
    variant) included."""
    import torch

    import paper_2506_03686_b200 as vp
    from paper_2506_03686_b200.api import execute_device

    dt = {1: torch.uint8, 2: torch.int16}[elem]
    n = int(np.prod(shape))
    seen = 0
    for jit in (True, False):
        prog = vp.build_program(vp.TensorLayout.from_shape(shape, elem), vp.from_numpy_convention(axes),
                                force="tile", jit=jit)
        vec = [ln for ln in prog.text.splitlines() if ln.startswith("vector elems")][0]
        seen += any(f", W {v}" in vec for v in (2, 4, 8)) and "residue" in vec and 16 // elem != int(vec.rsplit("W ", 1)[1].split()[0])
        x = torch.randint(0, 255, (n * elem,), dtype=torch.uint8, device="cuda")
        want = x.view(dt).view(shape).permute(axes).reshape(-1)
        assert torch.equal(execute_device(prog, x).view(dt).view(-1), want), (shape, jit)
        big = torch.randint(0, 255, (n * elem + elem,), dtype=torch.uint8, device="cuda")
        want2 = big[elem:].view(dt).view(shape).permute(axes).reshape(-1)
        assert torch.equal(execute_device(prog, big[elem:]).view(dt).view(-1), want2), (shape, jit, "misaligned src")
    assert seen >= 1, prog.text
