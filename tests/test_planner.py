"""Host-side planner and API algebra (no GPU needed).

Mirrors the reference's own unit tests for the same names
(/root/reference/pkg/tests/test_core.py, test_planner.py): merge results are
checked against the reference's merge_dimensions output recorded in the
golden file for all 1150 cases.
"""

from __future__ import annotations

import numpy as np
import pytest

import paper_2506_03686_b200 as vp
from paper_2506_03686_b200 import LayoutError, PermutationMap, TensorLayout
from tests.helpers import golden


# ------------------------------------------------------------ core algebra
def test_strides():
    assert vp.compute_strides((7, 5, 3)) == (1, 7, 35)          # test_core.py:45-48
    assert vp.compute_strides((4, 8, 16, 2)) == (1, 4, 32, 512)
    with pytest.raises(LayoutError):
        vp.compute_strides(())
    with pytest.raises(LayoutError):
        vp.compute_strides((4, 0, 2))


def test_permuted_layout_and_conventions():
    lay = TensorLayout((4, 8, 16, 2))
    assert vp.permuted_layout(lay, PermutationMap((3, 1, 2, 0))).shape_outer_first() == (4, 16, 8, 2)
    assert vp.to_numpy_convention(PermutationMap((2, 0, 1, 3))) == (0, 2, 3, 1)   # test_core.py:104-107
    rng = np.random.default_rng(1)
    for _ in range(50):
        n = int(rng.integers(1, 9))
        pm = PermutationMap(tuple(int(x) for x in rng.permutation(n)))
        assert vp.from_numpy_convention(vp.to_numpy_convention(pm)).sigma == pm.sigma
    with pytest.raises(LayoutError):
        PermutationMap((0, 0, 1))
    with pytest.raises(LayoutError):
        vp.permuted_layout(TensorLayout((2, 2)), PermutationMap((0, 1, 2)))
    with pytest.raises(LayoutError):
        TensorLayout((2, 2), 3)


def test_map_algebra():
    pm = PermutationMap((2, 0, 1))
    assert pm.compose(pm.inverse()).is_identity
    assert pm.dest_position(0) == 1


# ------------------------------------------------------------ merge (native planner)
def test_merge_matches_reference_on_all_golden_cases():
    """planner.py:211-241 semantics, compared with the reference's own output."""
    for c in golden()["cases"]:
        ml, mp = vp.merge_dimensions(TensorLayout(tuple(c["dims"]), c["elem"]), PermutationMap(tuple(c["sigma"])))
        assert list(ml.dims) == c["merged_dims"] and list(mp.sigma) == c["merged_sigma"], c["name"]


def test_merge_known_answers():
    # test_planner.py:24-52
    ml, mp = vp.merge_dimensions(TensorLayout((3, 5, 7)), PermutationMap((2, 0, 1)))
    assert ml.dims == (15, 7) and mp.sigma == (1, 0)
    ml, _ = vp.merge_dimensions(TensorLayout((9, 8, 4)), PermutationMap((2, 0, 1)))
    assert ml.dims == (72, 4)
    ml, mp = vp.merge_dimensions(TensorLayout((3, 4, 5)), PermutationMap((0, 1, 2)))
    assert ml.dims == (60,) and mp.sigma == (0,)
    ml, _ = vp.merge_dimensions(TensorLayout((3, 1, 5, 2)), PermutationMap((3, 0, 1, 2)))
    assert ml.dims == (15, 2)
    ml, mp = vp.merge_dimensions(TensorLayout((1, 1)), PermutationMap((1, 0)))
    assert ml.dims == (1,) and mp.sigma == (0,)


# ------------------------------------------------------------ classification
def _plan(shape, axes, elem=4, **kw):
    return vp.build_program(TensorLayout.from_shape(shape, elem), vp.from_numpy_convention(axes), **kw)


def test_classification_of_baseline_configs():
    from paper_2506_03686_b200.workloads import CONFIGS

    kinds = {k: _plan(w.shape, w.axes, w.elem_bytes).kernel for k, w in CONFIGS.items()}
    assert kinds == {"cfg1": "tile", "cfg2": "tile", "cfg3": "tile", "cfg4": "rows", "cfg5": "tile"}
    # merged forms
    assert _plan((32, 64, 56, 56), (0, 2, 3, 1)).merged_layout.dims == (3136, 64, 32)
    assert _plan((128, 64, 32, 512), (2, 0, 1, 3), 8).merged_layout.dims == (512, 32, 8192)
    assert _plan((17, 9, 13, 15, 11, 27), (5, 2, 0, 4, 1, 3)).merged_layout.rank == 6


def test_classification_edges():
    assert _plan((5, 7, 9), (0, 1, 2)).kernel in ("copy", "gather")           # identity
    assert _plan((50, 70, 90), (0, 1, 2)).kernel == "copy"
    assert _plan((8, 16, 3), (1, 0, 2)).kernel == "gather"                      # tiny
    assert _plan((640, 320, 3), (1, 0, 2)).kernel == "tile"                     # 12 B rows -> K3 tile
    assert _plan((64, 32, 1024), (1, 0, 2)).kernel == "rows"                    # 4 KiB rows -> K1
    assert _plan((1, 1), (1, 0)).kernel == "gather"


@pytest.mark.parametrize("elem", [1, 2, 4, 8, 16])
def test_tile_plan_invariants(elem):
    """Tiles fit the smem budget, cover the tensor, and runs are >= 1."""
    rng = np.random.default_rng(elem)
    for _ in range(60):
        rank = int(rng.integers(2, 7))
        shape = tuple(int(rng.integers(1, 40)) for _ in range(rank))
        axes = tuple(int(a) for a in rng.permutation(rank))
        p = _plan(shape, axes, elem, force="tile")
        m = p.metadata
        assert p.kernel == "tile"
        assert m["smem_bytes"] <= 227 * 1024
        assert m["tile_elems"] * m["num_tiles"] >= p.num_elements
        assert m["src_run"] >= 1 and m["dst_run"] >= 1
        assert m["tile_elems"] % m["src_run"] == 0 and m["tile_elems"] % m["dst_run"] == 0


def test_vectorisation_choices():
    p = _plan((4096, 4096), (1, 0))
    assert "vector elems: R 4, W 4" in p.text
    p = _plan((2,) * 20, tuple(np.random.default_rng(0).permutation(20).tolist()), 8)
    assert p.kernel == "tile"
    p = _plan((17, 9, 13, 15, 11, 27), (5, 2, 0, 4, 1, 3))
    # odd strides: runs start off 16-byte alignment -> aligned-superset reads
    assert "aligned supersets of misaligned runs" in p.text


def test_plan_cache_and_immutability():
    a = _plan((30, 40), (1, 0))
    b = _plan((30, 40), (1, 0))
    assert a is b
    with pytest.raises(Exception):
        a.kernel = "x"


def test_format_plan_mentions_key_facts():
    text = vp.format_plan(_plan((4096, 4096), (1, 0)))
    for key in ("kernel class", "merged dims", "tile elements", "smem pitch", "tiles:"):
        assert key in text


def test_machine_elem_width_mismatch_rejected():
    class M:
        elem_width = 8

    with pytest.raises(LayoutError):
        vp.build_program(TensorLayout((4, 4), 4), PermutationMap((1, 0)), M())


# ------------------------------------------------------------ per-case code generation
def test_emit_source_is_deterministic_and_specialised():
    """emit_source analog (emit.py:343-363): same plan -> same text; the
    TileParams block is baked in as constants."""
    p = _plan((4096, 4096), (1, 0))
    a = vp.emit_source(p)
    vp.program_cache_clear()
    b = vp.emit_source(_plan((4096, 4096), (1, 0)))
    assert a == b
    assert "vpg_tile_jit" in a and "#define VPG_JIT 1" in a and "vpg_kp[" in a
    assert vp.emit_source(_plan((17, 9, 13, 15, 11, 27), (5, 2, 0, 4, 1, 3))) != a
    with pytest.raises(LayoutError):
        vp.emit_source(_plan((128, 64, 32, 512), (2, 0, 1, 3), 8))     # rows plan: not specialised


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2", "cfg3", "cfg5"])
def test_specialised_kernels_compile_with_nvrtc(cfg):
    """The generated per-case sources compile for sm_100a (NVRTC, no GPU)."""
    from paper_2506_03686_b200.workloads import CONFIGS

    w = CONFIGS[cfg]
    vp.jit_compile(_plan(w.shape, w.axes, w.elem_bytes))


def test_scalar_w_kernels_declare_smem_alignment():
    """Specialised kernels with a scalar W walk declare the 128-byte
    alignment of the dynamic smem (VPG_SMEM_DECL, jit.cpp); V x V plans keep
    the computed base.  Both variants compile."""
    from paper_2506_03686_b200.workloads import CONFIGS

    w3, w1 = CONFIGS["cfg3"], CONFIGS["cfg1"]
    p3 = _plan(w3.shape, w3.axes, w3.elem_bytes)
    p1 = _plan(w1.shape, w1.axes, w1.elem_bytes)
    assert "W 1" in p3.text and "#define VPG_SMEM_DECL 1" in vp.emit_source(p3)
    assert "VxV" in p1.text and "#define VPG_SMEM_DECL" not in vp.emit_source(p1)
    # 1-byte misaligned transpose: scalar W walk through 32-bit registers
    p = _plan((203, 517), (1, 0), 1, force="tile")
    assert "#define VPG_SMEM_DECL 1" in vp.emit_source(p)
    vp.jit_compile(p)


def test_specialised_random_plans_compile():
    rng = np.random.default_rng(9)
    for elem in (1, 2, 4, 8, 16):
        rank = int(rng.integers(2, 6))
        shape = tuple(int(rng.integers(2, 30)) for _ in range(rank))
        axes = tuple(int(a) for a in rng.permutation(rank))
        vp.jit_compile(_plan(shape, axes, elem, force="tile"))


def test_tile_candidates_for_autotuning():
    """VPG_TILE_CANDIDATE(n): distinct tile shapes, each a complete plan;
    past the last candidate plan creation fails."""
    shapes = set()
    for c in range(6):
        p = _plan((64, 48, 80), (2, 0, 1), candidate=c)
        m = p.metadata
        assert p.kernel == "tile" and m["tile_elems"] * m["num_tiles"] >= p.num_elements
        shapes.add((m["src_run"], m["dst_run"], m["tile_elems"]))
    assert len(shapes) == 6
    assert _plan((64, 48, 80), (2, 0, 1), candidate=0).text == _plan((64, 48, 80), (2, 0, 1)).text
    with pytest.raises(LayoutError):
        _plan((6, 5), (1, 0), force="tile", candidate=200)


def test_dense_base_of_permuted_views():
    """permute() accepts permuted views of dense memory: the view is mapped
    back to its dense base and the axes are composed (host logic only)."""
    import torch

    from paper_2506_03686_b200.api import _dense_base

    base = torch.arange(6 * 1 * 10 * 12 * 7).reshape(6, 1, 10, 12, 7)
    rng = np.random.default_rng(4)
    for _ in range(200):
        p1 = tuple(int(a) for a in rng.permutation(5))
        p2 = tuple(int(a) for a in rng.permutation(5))
        v = base.permute(p1)
        b, ax = _dense_base(torch, v, p2)
        assert b.is_contiguous() and b.data_ptr() == base.data_ptr()
        assert torch.equal(b.permute(ax), v.permute(p2))
    with pytest.raises(LayoutError):
        _dense_base(torch, base[:, :, ::2], (0, 1, 2, 3, 4))


def test_baseline_layout_choices():
    """The layout each BASELINE config is planned with (kernels):
    cfg1/cfg2/cfg5 the 128-byte congruent swizzled rows with V x V W blocks,
    cfg3 residue row strides for its misaligned runs, TMA bulk reads for long
    runs that cannot take the congruent layout, and the
    cfg5 pull exchange at G = 8 keeping the 256 x 128 tile."""
    from paper_2506_03686_b200.sharded import _programs, fused_method
    from paper_2506_03686_b200.workloads import CONFIGS
    from tests.sim_tile import tile_params

    def tp(k):
        w = CONFIGS[k]
        return tile_params(_plan(w.shape, w.axes, w.elem_bytes)), _plan(w.shape, w.axes, w.elem_bytes)

    def tp_shape(shape, axes, e):
        p = _plan(shape, axes, e, force="tile")
        return tile_params(p), p

    for k in ("cfg1", "cfg2"):
        t, p = tp(k)
        # congruent rows, V x V W blocks, swizzle keyed on the 4-row group
        assert t.ph[0].swz == 3 and t.ph[1].swz == 3 and t.pitch == t.Ls and not t.bulk, k
        assert t.ph[1].w2 == 1 and t.ph[1].vrow == t.pitch, k
        assert "smem chunk swizzle" in p.text and "16-byte stores" in p.text
    t, p = tp("cfg3")
    # residue strides modulo 128 bytes (32 words); the bank model keeps them
    # unswizzled (W lanes: 2.5 wavefronts per access plain, 4.0 with the
    # address swizzle, whose XOR lands on the strides' own bank pattern)
    assert t.ph[0].rshift == 2 and t.rres == 31 and t.hmask == 0 and t.ph[0].swz == 0 and t.ph[1].swz == 0
    t, p = tp("cfg5")
    # 2 KiB power-of-two runs: congruent layout + V x V blocks (bulk reads
    # remain for long runs that cannot take it)
    assert t.bulk == 0 and t.ph[1].w2 == 1 and t.ph[0].swz == 2
    t, p = tp_shape((2, 3, 1000, 500), (0, 2, 1, 3), 8)        # 4000-byte runs: not a power of two
    assert t.bulk == 1 and "TMA bulk copy" in p.text
    w = CONFIGS["cfg5"]
    assert fused_method(w.shape, w.axes, 8, 2) == "push"
    assert fused_method(w.shape, w.axes, 8, 8) == "pull"
    (pp,) = _programs(w.shape, w.axes, 8, 8, [3], pull=True)
    t = tile_params(pp)
    assert t.pull == 1 and t.nshards == 8 and t.dst_bias == 3 * (w.numel // 8) and t.shard_shift == 25
    assert (pp.metadata["src_run"], pp.metadata["dst_run"]) == (256, 128)


def test_small_problem_tiles_and_groups():
    """Problems under 512 MiB get half-size tiles; separable thread groups
    leave ngroups == 1 (the specialised kernel unrolls the whole walk)."""
    from tests.sim_tile import tile_params

    big = tile_params(_plan((2,) * 28, tuple(int(a) for a in np.random.default_rng(0).permutation(28)), 8))
    small = tile_params(_plan((4096, 4096), (1, 0)))
    assert small.T * 4 <= 24 * 1024 + 8192 < big.T * 8 + 8192
    t = tile_params(_plan((17, 9, 13, 15, 11, 27), (5, 2, 0, 4, 1, 3)))
    assert t.ph[0].ngroups == 1 and t.ph[1].ngroups == 1
