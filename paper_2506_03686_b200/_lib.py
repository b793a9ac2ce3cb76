"""ctypes binding to libvpgpu.so (the C ABI in include/vpgpu.h).

The product path has no CPU fallback: if the library is missing the import
of any compute entry point raises immediately.
"""

from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
# VPG_LIB_PATH: development override (A/B of library builds, tools/); default in-tree
LIB_PATH = os.environ.get("VPG_LIB_PATH") or os.path.join(HERE, "libvpgpu.so")

VPG_OK, VPG_EINVAL, VPG_EUNSUPPORTED, VPG_ECUDA, VPG_ENOMEM = range(5)
KERNEL_NAMES = {0: "copy", 1: "rows", 2: "tile", 3: "gather"}
VPG_FORCE_GATHER = 0x1
VPG_FORCE_TILE = 0x2
VPG_NO_MERGE = 0x4
VPG_FORCE_JIT = 0x8
VPG_NO_JIT = 0x10
VPG_SHARD_PULL = 0x20
VPG_MAX_RANK = 64
VPG_MAX_SHARDS = 64
VPG_IPC_HANDLE_BYTES = 64


class ShardSync(ctypes.Structure):
    """vpg_shard_sync (include/vpgpu.h): device-side exchange ordering."""
    _fields_ = [("flags", ctypes.c_void_p * 64), ("epoch", ctypes.c_ulonglong), ("done_counter", ctypes.c_void_p)]

# symbols declared in include/vpgpu.h (checked by tests/test_abi.py)
EXPORTED = (
    "vpg_version",
    "vpg_last_error",
    "vpg_merge_dimensions",
    "vpg_plan_create",
    "vpg_plan_create_sharded",
    "vpg_permute",
    "vpg_permute_sharded",
    "vpg_permute_sharded_pull",
    "vpg_permute_sharded_sync",
    "vpg_permute_sharded_emulated",
    "vpg_ipc_export",
    "vpg_ipc_import",
    "vpg_ipc_release",
    "vpg_permute_host",
    "vpg_permute_host_async",
    "vpg_permute_host_bounded",
    "vpg_permute_nd",
    "vpg_plan_info_get",
    "vpg_plan_describe",
    "vpg_plan_emit_source",
    "vpg_plan_jit_compile",
    "vpg_plan_tile_params",
    "vpg_plan_destroy",
)


class PlanInfo(ctypes.Structure):
    _fields_ = [
        ("kernel_class", ctypes.c_int32),
        ("elem_bytes", ctypes.c_int32),
        ("rank", ctypes.c_int32),
        ("dims", ctypes.c_int64 * VPG_MAX_RANK),
        ("sigma", ctypes.c_int32 * VPG_MAX_RANK),
        ("num_elements", ctypes.c_int64),
        ("tile_elems", ctypes.c_int64),
        ("src_run", ctypes.c_int64),
        ("dst_run", ctypes.c_int64),
        ("num_tiles", ctypes.c_int64),
        ("smem_pitch", ctypes.c_int32),
        ("smem_bytes", ctypes.c_int32),
        ("vec_elems", ctypes.c_int32),
        ("threads", ctypes.c_int32),
        ("grid_hint", ctypes.c_int64),
        ("predicted_efficiency", ctypes.c_double),
        ("host_chunks", ctypes.c_int32),
        ("jit_state", ctypes.c_int32),
        ("shards", ctypes.c_int32),
        ("shard_index", ctypes.c_int32),
    ]


_lib = None
_lock = threading.Lock()


class LibraryMissing(RuntimeError):
    pass


def lib():
    """Load libvpgpu.so (once).  Raises LibraryMissing if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise LibraryMissing(
                f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                "or `make -C paper_2506_03686_b200/csrc` (there is no CPU fallback)"
            )
        L = ctypes.CDLL(LIB_PATH)
        i64p = ctypes.POINTER(ctypes.c_int64)
        i32p = ctypes.POINTER(ctypes.c_int32)
        vp = ctypes.c_void_p
        L.vpg_version.restype = ctypes.c_int
        L.vpg_last_error.restype = ctypes.c_char_p
        L.vpg_merge_dimensions.argtypes = [ctypes.c_int, i64p, i32p, ctypes.POINTER(ctypes.c_int), i64p, i32p]
        L.vpg_plan_create.argtypes = [ctypes.c_int, i64p, i32p, ctypes.c_int, ctypes.c_uint,
                                      ctypes.POINTER(vp)]
        L.vpg_plan_create_sharded.argtypes = [ctypes.c_int, i64p, i32p, ctypes.c_int, ctypes.c_uint,
                                              ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp)]
        L.vpg_permute.argtypes = [vp, vp, vp, vp]
        L.vpg_permute_sharded.argtypes = [vp, vp, ctypes.POINTER(vp), vp]
        L.vpg_permute_sharded_pull.argtypes = [vp, ctypes.POINTER(vp), vp, vp]
        L.vpg_permute_sharded_sync.argtypes = [vp, ctypes.POINTER(vp), ctypes.POINTER(vp), vp, vp]
        L.vpg_permute_sharded_emulated.argtypes = [ctypes.POINTER(vp), ctypes.c_int, ctypes.POINTER(vp),
                                                   ctypes.POINTER(vp), vp]
        L.vpg_ipc_export.argtypes = [vp, vp, ctypes.POINTER(ctypes.c_uint64)]
        L.vpg_ipc_import.argtypes = [vp, ctypes.c_uint64, ctypes.POINTER(vp)]
        L.vpg_ipc_release.argtypes = [vp]
        L.vpg_permute_host.argtypes = [vp, vp, vp, vp, vp, vp]
        L.vpg_permute_host_async.argtypes = [vp, vp, vp, vp, vp, vp]
        L.vpg_permute_host_bounded.argtypes = [vp, vp, vp, vp, ctypes.c_size_t, vp]
        L.vpg_permute_nd.argtypes = [ctypes.c_int, i64p, i32p, ctypes.c_int, vp, vp, vp]
        L.vpg_plan_info_get.argtypes = [vp, ctypes.POINTER(PlanInfo)]
        L.vpg_plan_describe.argtypes = [vp, ctypes.c_char_p, ctypes.c_size_t]
        L.vpg_plan_emit_source.argtypes = [vp, ctypes.c_char_p, ctypes.c_size_t]
        L.vpg_plan_jit_compile.argtypes = [vp]
        L.vpg_plan_tile_params.argtypes = [vp, vp, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]
        L.vpg_plan_destroy.argtypes = [vp]
        L.vpg_plan_destroy.restype = None
        for name in ("vpg_merge_dimensions", "vpg_plan_create", "vpg_permute", "vpg_permute_host",
                     "vpg_plan_create_sharded", "vpg_permute_sharded", "vpg_permute_sharded_pull",
                     "vpg_permute_sharded_sync", "vpg_permute_sharded_emulated", "vpg_ipc_export", "vpg_ipc_import",
                     "vpg_ipc_release",
                     "vpg_permute_host_async", "vpg_permute_host_bounded",
                     "vpg_permute_nd", "vpg_plan_info_get", "vpg_plan_describe", "vpg_plan_emit_source",
                     "vpg_plan_jit_compile", "vpg_plan_tile_params"):
            getattr(L, name).restype = ctypes.c_int
        _lib = L
        return L


def last_error() -> str:
    msg = lib().vpg_last_error()
    return msg.decode() if msg else ""


def arrays(dims, sigma):
    rank = len(dims)
    d = (ctypes.c_int64 * max(rank, 1))(*[int(x) for x in dims])
    s = (ctypes.c_int32 * max(rank, 1))(*[int(x) for x in sigma])
    return rank, d, s
