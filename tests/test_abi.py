"""The C-ABI library loads and exports every symbol include/vpgpu.h declares;
host-only entry points (planning, merge, describe, errors) work without a GPU."""

from __future__ import annotations

import ctypes
import os
import re
import subprocess

import pytest

from paper_2506_03686_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "vpgpu.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(vpg_[a-z_]+)\s*\(", text)))


def test_header_declares_the_python_binding_list():
    assert declared_symbols() == sorted(_lib.EXPORTED)


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    for name in declared_symbols():
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (vpg_[a-z_]+)", out))
    assert set(declared_symbols()) <= exported


def test_version_and_last_error():
    L = _lib.lib()
    assert L.vpg_version() == 6
    rank, d, s = _lib.arrays((3, 2), (0, 0))
    p = ctypes.c_void_p()
    assert L.vpg_plan_create(rank, d, s, 4, 0, ctypes.byref(p)) == _lib.VPG_EINVAL
    assert "bijection" in _lib.last_error()
    rank, d, s = _lib.arrays((3, 2), (1, 0))
    assert L.vpg_plan_create(rank, d, s, 3, 0, ctypes.byref(p)) == _lib.VPG_EINVAL
    assert "element width" in _lib.last_error()
    rank, d, s = _lib.arrays((3, 0), (1, 0))
    assert L.vpg_plan_create(rank, d, s, 4, 0, ctypes.byref(p)) == _lib.VPG_EINVAL


def test_plan_info_and_describe_host_only():
    L = _lib.lib()
    rank, d, s = _lib.arrays((4096, 4096), (1, 0))
    p = ctypes.c_void_p()
    assert L.vpg_plan_create(rank, d, s, 4, 0, ctypes.byref(p)) == 0
    info = _lib.PlanInfo()
    assert L.vpg_plan_info_get(p, ctypes.byref(info)) == 0
    assert info.kernel_class == 2 and info.rank == 2 and info.num_elements == 4096 * 4096
    assert info.tile_elems * info.num_tiles >= info.num_elements
    buf = ctypes.create_string_buffer(4096)
    assert L.vpg_plan_describe(p, buf, 4096) == 0
    assert b"tile" in buf.value
    L.vpg_plan_destroy(p)


def test_null_arguments_rejected():
    L = _lib.lib()
    assert L.vpg_plan_create(1, None, None, 4, 0, None) == _lib.VPG_EINVAL
    assert L.vpg_permute(None, None, None, None) == _lib.VPG_EINVAL
    assert L.vpg_plan_describe(None, None, 0) == _lib.VPG_EINVAL


def test_product_has_no_cpu_fallback(monkeypatch):
    """Without the native library the API raises instead of computing on CPU."""
    import paper_2506_03686_b200 as vp

    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", "/nonexistent/libvpgpu.so")
    vp.program_cache_clear()
    with pytest.raises(_lib.LibraryMissing):
        vp.build_program(vp.TensorLayout((3, 2)), vp.PermutationMap((1, 0)))


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2506_03686_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f


def test_sharded_plan_errors_without_gpu():
    """Sharded plans are created host-side; bad shard arguments and
    non-sharding shapes fail with the documented statuses."""
    import ctypes

    L = _lib.lib()
    rank, d, s = _lib.arrays((4, 8), (1, 0))
    p = ctypes.c_void_p()
    assert L.vpg_plan_create_sharded(rank, d, s, 4, 0, 2, 2, ctypes.byref(p)) == _lib.VPG_EINVAL
    assert L.vpg_plan_create_sharded(rank, d, s, 4, 0, 0, 0, ctypes.byref(p)) == _lib.VPG_EINVAL
    assert L.vpg_plan_create_sharded(rank, d, s, 4, 0, 3, 0, ctypes.byref(p)) == _lib.VPG_EUNSUPPORTED
    assert "cannot shard" in _lib.last_error()
    rank, d, s = _lib.arrays((32, 16), (1, 0))
    assert L.vpg_plan_create_sharded(rank, d, s, 4, 0, 2, 1, ctypes.byref(p)) == _lib.VPG_OK
    # ordinary entry points refuse a sharded plan
    assert L.vpg_permute(p, ctypes.c_void_p(16), ctypes.c_void_p(4096), None) == _lib.VPG_EINVAL
    assert "vpg_permute_sharded" in _lib.last_error()
    L.vpg_plan_destroy(p)


def test_rank_above_64_with_unit_dims_is_accepted():
    """Size-1 dims are dropped before the rank limit (the reference has no
    rank cap, core.py:58-88; merge_dimensions drops them, planner.py:222-227)."""
    import numpy as np

    from paper_2506_03686_b200 import PermutationMap, TensorLayout, build_program, merge_dimensions

    rng = np.random.default_rng(7)
    dims = [1] * 70
    for k, e in zip(rng.choice(70, 5, replace=False), (3, 5, 2, 7, 4)):
        dims[k] = int(e)
    sigma = tuple(int(v) for v in rng.permutation(70))
    lay, pm = TensorLayout(tuple(dims), 4), PermutationMap(sigma)
    ml, mp = merge_dimensions(lay, pm)
    assert 1 <= ml.rank <= 5 and np.prod(ml.dims) == 3 * 5 * 2 * 7 * 4
    prog = build_program(lay, pm)
    assert prog.num_elements == 3 * 5 * 2 * 7 * 4
    # 70 dims that are not size 1 stay out of range
    with pytest.raises(ValueError):
        build_program(TensorLayout((2,) * 70, 4), PermutationMap(tuple(range(70))[::-1]))


def test_overlapping_buffers_rejected_before_any_device_work():
    L = _lib.lib()
    rank, d, s = _lib.arrays((64, 48), (1, 0))
    p = ctypes.c_void_p()
    assert L.vpg_plan_create(rank, d, s, 4, 0, ctypes.byref(p)) == 0
    base = 1 << 40
    # partial overlap (dst starts inside src): EINVAL, no launch attempted
    assert L.vpg_permute(p, ctypes.c_void_p(base), ctypes.c_void_p(base + 256), None) == _lib.VPG_EINVAL
    assert "overlap" in _lib.last_error()
    assert L.vpg_permute(p, ctypes.c_void_p(base + 256), ctypes.c_void_p(base), None) == _lib.VPG_EINVAL
    L.vpg_plan_destroy(p)
