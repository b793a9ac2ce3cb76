"""Public plan / permute API -- the drop-in for vecperm's hot path.

Reference boundary (pkg/src/vecperm/__init__.py:3-34; README "Library in
five lines"):

    ir = build_program(layout, pmap, machine)        # ir.py:441-456
    out, counters = execute(ir, input_buf)           # vm.py:105-110

Here ``build_program`` calls the native planner in libvpgpu.so (merge +
classify + tile selection) and returns an immutable :class:`GpuProgram`;
``execute`` runs it on the B200 through the C ABI.  ``permute(x, axes)`` is
the torch-convention convenience (``out = x.permute(axes).contiguous()``).

There is no CPU fallback: every element move is a CUDA kernel launch in
libvpgpu.so; host buffers given to ``execute`` are staged through device
memory (that is the end-to-end path the bench times).
"""

from __future__ import annotations

import ctypes
import os
import functools
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .core import (
    LayoutError,
    PermutationMap,
    TensorLayout,
    from_numpy_convention,
    permuted_layout,
)

__all__ = [
    "GpuTarget",
    "GpuProgram",
    "VpgError",
    "merge_dimensions",
    "build_program",
    "execute",
    "permute",
    "format_plan",
    "emit_source",
    "jit_compile",
    "program_cache_clear",
    "autotune",
    "build_sharded_program",
    "launch_sharded",
    "release_scratch",
]


class VpgError(RuntimeError):
    """CUDA-side failure (VPG_ECUDA / VPG_ENOMEM)."""


def _check(status: int, what: str):
    if status == _lib.VPG_OK:
        return
    msg = f"{what}: {_lib.last_error()}"
    if status in (_lib.VPG_EINVAL,):
        raise LayoutError(msg)
    if status == _lib.VPG_EUNSUPPORTED:
        raise LayoutError("unsupported: " + msg)
    raise VpgError(msg)


def _measured_hbm_gbs(default: float = 6555.2) -> float:
    """HBM copy bandwidth (read+write GB/s) from the driver-written
    MEASURED_PEAKS.json at the repo root, when present."""
    import json
    import os

    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"])
    except (OSError, ValueError, KeyError, TypeError):
        return default


@dataclass(frozen=True)
class GpuTarget:
    """GPU target descriptor (the MachineConfig analog, machine.py:13-40).

    The planner is device-agnostic (plans are POD kernel arguments); the
    descriptor records what the numbers in DESIGN.md assume.
    """

    name: str = "B200"
    arch: str = "sm_100a"
    sms: int = 148
    smem_per_sm: int = 228 * 1024
    hbm_gbs: float = field(default_factory=_measured_hbm_gbs)   # MEASURED_PEAKS.json (copy, read+write)


# ------------------------------------------------------------------ merge
def merge_dimensions(layout: TensorLayout, pmap: PermutationMap):
    """Fuse adjacent dims whose adjacency and order survive the map.

    Same contract as planner.py:211-241 (size-1 dims dropped first; the
    element bijection is preserved); computed by the native planner.
    """
    if pmap.rank != layout.rank:
        raise LayoutError("map rank does not match layout rank")
    L = _lib.lib()
    rank, d, s = _lib.arrays(layout.dims, pmap.sigma)
    od = (ctypes.c_int64 * rank)()
    os_ = (ctypes.c_int32 * rank)()
    orank = ctypes.c_int(0)
    _check(L.vpg_merge_dimensions(rank, d, s, ctypes.byref(orank), od, os_), "merge_dimensions")
    r = orank.value
    return TensorLayout(tuple(od[:r]), layout.elem_width), PermutationMap(tuple(os_[:r]))


# ------------------------------------------------------------------ program
class _Handle:
    """Owns one vpg_plan*; destroyed with the program."""

    __slots__ = ("ptr",)

    def __init__(self, ptr):
        self.ptr = ptr

    def __del__(self):
        try:
            if self.ptr:
                _lib.lib().vpg_plan_destroy(self.ptr)
                self.ptr = None
        except Exception:
            pass


@dataclass(frozen=True)
class GpuProgram:
    """Immutable, shareable plan (the IRProgram analog, ir.py:96-108)."""

    layout: TensorLayout
    pmap: PermutationMap
    merged_layout: TensorLayout
    merged_pmap: PermutationMap
    kernel: str
    metadata: dict = field(compare=False)
    text: str = field(compare=False)
    _handle: _Handle = field(compare=False, repr=False)

    @property
    def num_elements(self) -> int:
        return self.layout.num_elements

    @property
    def out_layout(self) -> TensorLayout:
        return permuted_layout(self.layout, self.pmap)

    @functools.cached_property
    def out_shape(self) -> tuple:
        """Output shape, NumPy/torch order (outer-first)."""
        return self.out_layout.shape_outer_first()

    @property
    def nbytes(self) -> int:
        return self.layout.num_elements * self.layout.elem_width

    @property
    def algorithmic_bytes(self) -> int:
        """One read + one write per element."""
        return 2 * self.nbytes

    @property
    def handle(self) -> int:
        return self._handle.ptr

    @property
    def jit_state(self) -> int:
        """0: ahead-of-time kernel, 1: specialisation pending (first launch
        compiles it), 2: NVRTC-specialised kernel loaded, -1: failed."""
        info = _lib.PlanInfo()
        _check(_lib.lib().vpg_plan_info_get(self.handle, ctypes.byref(info)), "plan_info")
        return info.jit_state


_cache: dict = {}
_cache_lock = threading.Lock()


def program_cache_clear():
    with _cache_lock:
        _cache.clear()


def _wrap(ptr, layout: TensorLayout, pmap: PermutationMap) -> "GpuProgram":
    """GpuProgram around a freshly created plan handle."""
    L = _lib.lib()
    handle = _Handle(ptr)
    info = _lib.PlanInfo()
    _check(L.vpg_plan_info_get(ptr, ctypes.byref(info)), "plan_info")
    buf = ctypes.create_string_buffer(4096)
    _check(L.vpg_plan_describe(ptr, buf, 4096), "plan_describe")
    r = info.rank
    merged_layout = TensorLayout(tuple(info.dims[:r]), layout.elem_width)
    merged_pmap = PermutationMap(tuple(info.sigma[:r]))
    kernel = _lib.KERNEL_NAMES[info.kernel_class]
    meta = {
        "kernel": kernel,
        "merged_dims": merged_layout.dims,
        "merged_sigma": merged_pmap.sigma,
        "tile_elems": info.tile_elems,
        "src_run": info.src_run,
        "dst_run": info.dst_run,
        "num_tiles": info.num_tiles,
        "smem_pitch": info.smem_pitch,
        "smem_bytes": info.smem_bytes,
        "vec_elems": info.vec_elems,
        "threads": info.threads,
        "grid_hint": info.grid_hint,
        "predicted_efficiency": info.predicted_efficiency,
        "host_chunks": info.host_chunks,
        "shards": info.shards,
        "shard_index": info.shard_index,
        "source_shape": layout.dims,
        "source_map": pmap.sigma,
    }
    return GpuProgram(layout, pmap, merged_layout, merged_pmap, kernel, meta, buf.value.decode(), handle)


def build_program(layout: TensorLayout, pmap: PermutationMap, machine=None, merge: bool = True,
                  opt: bool = True, force: str | None = None, jit: bool | None = None,
                  candidate: int | None = None, tune: bool = False, _auto: bool = True) -> GpuProgram:
    """Plan a permutation (ir.py:441-456 signature; ``machine``/``opt`` kept
    for drop-in compatibility).

    ``force`` pins a kernel class for tests: ``"tile"`` or ``"gather"``.
    ``jit`` pins the per-case NVRTC specialisation of tile plans on/off
    (default: on for tensors of 4 MiB and more).
    ``candidate`` picks the n-th best tile shape of the cost model (tile
    plans; LayoutError past the last one).
    ``tune`` times the best few tile candidates on the current GPU and keeps
    the fastest (measured planning, like FFTW_MEASURE): the tuned program
    then answers later calls with the same arguments and ``tune=False``.
    ``VPG_TUNE=1`` in the environment does this for every tile plan of
    16 MiB and more (on random shapes it lifts the 10th-percentile
    fraction of copy from ~0.73 to ~0.80, tools/perf_sweep.py).
    """
    if _auto and not tune and candidate is None and os.environ.get("VPG_TUNE") == "1":
        # process-wide measured planning for large tile plans (needs a GPU)
        base = build_program(layout, pmap, machine, merge, opt, force, jit, _auto=False)
        if base.kernel == "tile" and base.nbytes >= (16 << 20) and not base.metadata.get("tuned_ms"):
            torch = _torch()
            if torch.cuda.is_available():
                return autotune(layout, pmap, merge=merge, force=force, jit=jit, candidates=6, reps=3)
        return base
    if tune:
        return autotune(layout, pmap, merge=merge, force=force, jit=jit)
    if pmap.rank != layout.rank:
        raise LayoutError("map rank does not match layout rank")
    if machine is not None and hasattr(machine, "elem_width") and machine.elem_width != layout.elem_width:
        raise LayoutError("layout and machine element widths differ")   # planner.py:307-308
    flags = 0
    if not merge:
        flags |= _lib.VPG_NO_MERGE
    if force == "tile":
        flags |= _lib.VPG_FORCE_TILE
    elif force == "gather":
        flags |= _lib.VPG_FORCE_GATHER
    elif force is not None:
        raise ValueError(f"unknown force={force!r}")
    if jit is True:
        flags |= _lib.VPG_FORCE_JIT
    elif jit is False:
        flags |= _lib.VPG_NO_JIT
    if candidate is not None:
        if not 0 <= candidate < 255:
            raise ValueError(f"candidate {candidate} out of range")
        flags |= ((candidate + 1) & 0xFF) << 8
    key = (layout.dims, layout.elem_width, pmap.sigma, flags)
    with _cache_lock:
        hit = _cache.get(key)
    if hit is not None:
        return hit
    L = _lib.lib()
    rank, d, s = _lib.arrays(layout.dims, pmap.sigma)
    ptr = ctypes.c_void_p()
    _check(L.vpg_plan_create(rank, d, s, layout.elem_width, flags, ctypes.byref(ptr)), "build_program")
    prog = _wrap(ptr, layout, pmap)
    with _cache_lock:
        _cache.setdefault(key, prog)
        return _cache[key]


def build_sharded_program(layout: TensorLayout, pmap: PermutationMap, shards: int, shard_index: int,
                          jit: bool | None = None, candidate: int | None = None, pull: bool = False) -> GpuProgram:
    """Plan of the fused sharded exchange (vpg_plan_create_sharded).

    push (default): the plan of input shard ``shard_index`` -- ONE tile
    kernel that reads the local input shard and stores every tile straight
    into the output shard that owns it.  pull: the plan of OUTPUT shard
    ``shard_index`` -- ONE tile kernel that reads its tiles' source runs from
    every input shard (peer memory) and writes the local output shard.
    Raises LayoutError when the shapes do not shard or no tile avoids the
    shard-indexing dims (callers then use the all-to-all path)."""
    if pmap.rank != layout.rank:
        raise LayoutError("map rank does not match layout rank")
    if not 1 <= shards <= _lib.VPG_MAX_SHARDS:
        raise LayoutError(f"shards must be in 1..{_lib.VPG_MAX_SHARDS}")
    flags = 0
    if jit is True:
        flags |= _lib.VPG_FORCE_JIT
    elif jit is False:
        flags |= _lib.VPG_NO_JIT
    if candidate is not None:
        flags |= ((candidate + 1) & 0xFF) << 8
    if pull:
        flags |= _lib.VPG_SHARD_PULL
    key = ("sharded", layout.dims, layout.elem_width, pmap.sigma, flags, shards, shard_index)
    with _cache_lock:
        hit = _cache.get(key)
    if hit is not None:
        return hit
    L = _lib.lib()
    rank, d, s = _lib.arrays(layout.dims, pmap.sigma)
    ptr = ctypes.c_void_p()
    _check(L.vpg_plan_create_sharded(rank, d, s, layout.elem_width, flags, shards, shard_index,
                                     ctypes.byref(ptr)), "build_sharded_program")
    prog = _wrap(ptr, layout, pmap)
    prog.metadata["pull"] = bool(pull)
    with _cache_lock:
        _cache.setdefault(key, prog)
        return _cache[key]


def launch_sharded_pull(program: GpuProgram, src_ptrs, dst_ptr: int, stream_ptr) -> None:
    """Enqueue the pull exchange kernel of one output shard
    (vpg_permute_sharded_pull): ``src_ptrs[q]`` = input shard q's buffer as
    seen from this device, ``dst_ptr`` = the local output shard."""
    G = program.metadata["shards"]
    if len(src_ptrs) != G:
        raise LayoutError(f"expected {G} source shards, got {len(src_ptrs)}")
    arr = (ctypes.c_void_p * G)(*[int(p) for p in src_ptrs])
    st = _lib.lib().vpg_permute_sharded_pull(program.handle, arr, ctypes.c_void_p(dst_ptr), stream_ptr)
    _check(st, "permute_sharded_pull")


def launch_sharded(program: GpuProgram, src_ptr: int, dst_ptrs, stream_ptr) -> None:
    """Enqueue the exchange kernel of one input shard (vpg_permute_sharded):
    ``dst_ptrs[q]`` = output shard q's buffer as seen from this device."""
    G = program.metadata["shards"]
    if len(dst_ptrs) != G:
        raise LayoutError(f"expected {G} destination shards, got {len(dst_ptrs)}")
    arr = (ctypes.c_void_p * G)(*[int(p) for p in dst_ptrs])
    st = _lib.lib().vpg_permute_sharded(program.handle, ctypes.c_void_p(src_ptr), arr, stream_ptr)
    _check(st, "permute_sharded")


def launch_sharded_sync(program: GpuProgram, src_ptrs, dst_ptrs, sync, stream_ptr) -> None:
    """Enqueue one rank's fused-exchange kernel with device-side ordering
    (vpg_permute_sharded_sync; ``sync`` an _lib.ShardSync or None).  Push
    plans: src_ptrs = [own input], dst_ptrs = every output shard; pull
    plans: src_ptrs = every input shard, dst_ptrs = [own output]."""
    arr_s = (ctypes.c_void_p * len(src_ptrs))(*[int(p) for p in src_ptrs])
    arr_d = (ctypes.c_void_p * len(dst_ptrs))(*[int(p) for p in dst_ptrs])
    st = _lib.lib().vpg_permute_sharded_sync(program.handle, arr_s, arr_d,
                                             ctypes.byref(sync) if sync is not None else None, stream_ptr)
    _check(st, "permute_sharded_sync")


def launch_sharded_emulated(programs, src_ptrs, dst_ptrs, stream_ptr) -> None:
    """Every rank's exchange kernel in one cooperative launch on this device,
    with the device-side exchange ordering between them
    (vpg_permute_sharded_emulated); returns once the step has finished."""
    G = len(programs)
    hs = [p.handle for p in programs]
    plans = (ctypes.c_void_p * G)(*[h.value if isinstance(h, ctypes.c_void_p) else h for h in hs])
    arr_s = (ctypes.c_void_p * G)(*[int(p) for p in src_ptrs])
    arr_d = (ctypes.c_void_p * G)(*[int(p) for p in dst_ptrs])
    _check(_lib.lib().vpg_permute_sharded_emulated(plans, G, arr_s, arr_d, stream_ptr), "permute_sharded_emulated")


def _time_program(torch, program, src, dst, flush, reps):
    """Median device time (ms) of one launch after an L2 flush."""
    stream = torch.cuda.current_stream(src.device)
    sp = ctypes.c_void_p(stream.cuda_stream)
    times = []
    for i in range(reps + 2):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        _launch(program, src.data_ptr(), dst.data_ptr(), sp)
        b.record(stream)
        b.synchronize()
        if i >= 2:                       # first launches compile/load the kernel
            times.append(a.elapsed_time(b))
    times.sort()
    return times[len(times) // 2]


def autotune(layout: TensorLayout, pmap: PermutationMap, candidates: int = 10, reps: int = 5,
             merge: bool = True, force: str | None = None, jit: bool | None = None,
             device=None, src=None, dst=None) -> GpuProgram:
    """Time the ``candidates`` best tile shapes of the cost model on the GPU
    and cache the fastest as the program for these arguments.  Non-tile
    plans are returned unchanged.  Needs a GPU (raises on CPU) and, while it
    runs, two scratch buffers of the tensor's size plus a 256 MiB L2-flush
    buffer; pass the CUDA tensors the program will run on as ``src``/``dst``
    to time on them instead (their contents are overwritten: ``dst`` only)."""
    base = build_program(layout, pmap, merge=merge, force=force, jit=jit, _auto=False)
    if base.kernel != "tile" or base.num_elements == 0:
        return base
    torch = _torch()
    if not torch.cuda.is_available():
        raise VpgError("autotune needs a CUDA device")
    if src is not None:
        dev = src.device
    else:
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    with torch.cuda.device(dev):
        if src is None:
            src = torch.empty(base.nbytes, dtype=torch.uint8, device=dev)
        if dst is None:
            dst = torch.empty(base.nbytes, dtype=torch.uint8, device=dev)
        for t in (src, dst):
            if not t.is_cuda or t.numel() * t.element_size() != base.nbytes or not t.is_contiguous():
                raise LayoutError("autotune buffers must be contiguous CUDA tensors of the tensor's size")
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        best, best_t = base, _time_program(torch, base, src, dst, flush, reps)
        for c in range(1, candidates):
            try:
                prog = build_program(layout, pmap, merge=merge, force=force, jit=jit, candidate=c)
            except LayoutError:
                break                     # fewer candidates than asked for
            t = _time_program(torch, prog, src, dst, flush, reps)
            if t < best_t:
                best, best_t = prog, t
        del src, dst, flush
    with _cache_lock:
        for k, v in list(_cache.items()):
            if v is base:
                _cache[k] = best
    best.metadata["tuned_ms"] = best_t
    return best


def emit_source(program: GpuProgram) -> str:
    """CUDA source of the program's specialised kernel (the reference's
    emit_source, emit.py:343-363).  Tile programs only."""
    L = _lib.lib()
    buf = ctypes.create_string_buffer(1 << 16)
    _check(L.vpg_plan_emit_source(program.handle, buf, len(buf)), "emit_source")
    return buf.value.decode()


def jit_compile(program: GpuProgram) -> None:
    """Compile the specialised kernel with NVRTC without a GPU (raises
    LayoutError with the NVRTC log on failure)."""
    _check(_lib.lib().vpg_plan_jit_compile(program.handle), "jit_compile")


def format_plan(program: GpuProgram) -> str:
    """Human-readable plan dump (format_plan analog, planner.py:386-419)."""
    return program.text


# ------------------------------------------------------------------ execute
def _torch():
    import torch

    return torch


def _stream_ptr(torch, device, stream):
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return ctypes.c_void_p(stream.cuda_stream)


def _launch(program: GpuProgram, src_ptr: int, dst_ptr: int, stream_ptr) -> None:
    st = _lib.lib().vpg_permute(program.handle, ctypes.c_void_p(src_ptr), ctypes.c_void_p(dst_ptr), stream_ptr)
    _check(st, "permute")


def _counters(program: GpuProgram) -> dict:
    c = dict(program.metadata)
    c["launches"] = 1 if program.num_elements > 0 else 0
    c["bytes_read"] = program.nbytes
    c["bytes_written"] = program.nbytes
    return c


def execute_device(program: GpuProgram, x, out=None, stream=None):
    """Permute a CUDA tensor (any dtype whose itemsize is the element width).

    Returns a tensor shaped like the output layout (outer-first)."""
    torch = _torch()
    if not isinstance(x, torch.Tensor) or not x.is_cuda:
        raise LayoutError("execute_device needs a CUDA tensor")
    es = x.element_size()
    nbytes = program.nbytes
    if es != program.layout.elem_width and not (x.dtype == torch.uint8 and x.numel() == nbytes):
        raise LayoutError(f"tensor itemsize {es} != element width {program.layout.elem_width}")
    if x.numel() * es != nbytes:
        raise LayoutError(f"tensor holds {x.numel()} elements, program expects {program.num_elements}")
    if not x.is_contiguous():
        raise LayoutError("input tensor must be contiguous (dense layout)")
    if out is None:
        if es == program.layout.elem_width:
            out = torch.empty(program.out_shape, dtype=x.dtype, device=x.device)
        else:
            out = torch.empty(nbytes, dtype=torch.uint8, device=x.device)
    else:
        if not out.is_cuda or not out.is_contiguous() or out.numel() * out.element_size() != nbytes:
            raise LayoutError("out must be a contiguous CUDA tensor of the output size")
        if out.device != x.device:
            raise LayoutError("out must be on the input's device")
    if program.num_elements == 0:
        return out
    xp, op = x.data_ptr(), out.data_ptr()
    if xp < op + nbytes and op < xp + nbytes:
        raise LayoutError("out-of-place only: out overlaps the input")
    dev = x.get_device()
    if stream is None:
        stream = torch.cuda.current_stream(dev)
    if dev != torch.cuda.current_device():
        with torch.cuda.device(dev):
            _launch(program, xp, op, ctypes.c_void_p(stream.cuda_stream))
    else:
        _launch(program, xp, op, ctypes.c_void_p(stream.cuda_stream))
    return out


def execute(program: GpuProgram, input_buf, trace: bool = False, out=None, stream=None, blocking: bool = True,
            max_device_bytes: int | None = None):
    """Run a program; returns ``(output, counters)`` like vm.py:105-110.

    * CUDA tensor input -> CUDA output tensor (outer-first output shape).
    * numpy array / bytes / CPU tensor input -> staged through device memory
      (chunked H2D / kernel / D2H pipeline); returns a flat numpy array of
      opaque words (``program.layout.dtype``) like the reference, or a CPU
      tensor for a CPU-tensor input.
    * ``blocking=False`` (pinned CPU tensors with ``out`` given): enqueue and
      return at once; consecutive calls overlap their transfers.  Call
      ``stream.synchronize()`` (default: the current stream) before reading
      ``out``.
    * Host tensors larger than the device can stage (or ``max_device_bytes``
      below twice the tensor): streamed through that much device scratch in
      chunks (vpg_permute_host_bounded; blocking).
    """
    torch = _torch()
    if isinstance(input_buf, torch.Tensor) and input_buf.is_cuda:
        res = execute_device(program, input_buf, out=out, stream=stream)
        return res, _counters(program)
    return (_execute_host(program, input_buf, out=out, stream=stream, blocking=blocking,
                          max_device_bytes=max_device_bytes), _counters(program))


_scratch: "collections.OrderedDict" = None      # (id(program), device) -> (program, d_in, d_out), LRU
_scratch_lock = threading.Lock()
SCRATCH_PROGRAMS = 4        # host-path programs whose device staging buffers stay cached


def _host_scratch(torch, program, dev):
    """Device staging buffers of the host path, kept per (program, device)
    for the last SCRATCH_PROGRAMS programs; the library orders reuse across
    in-flight calls.  An evicted pair is released only after the device has
    finished every call that may still use it (the library's internal
    streams are not known to torch's allocator)."""
    import collections

    global _scratch
    key = (id(program), dev.index)
    with _scratch_lock:
        if _scratch is None:
            _scratch = collections.OrderedDict()
        hit = _scratch.get(key)
        if hit is None or hit[0] is not program:
            hit = (program, torch.empty(program.nbytes, dtype=torch.uint8, device=dev),
                   torch.empty(program.nbytes, dtype=torch.uint8, device=dev))
            _scratch[key] = hit
        _scratch.move_to_end(key)
        if len(_scratch) > SCRATCH_PROGRAMS:
            for d in {k[1] for k in _scratch}:
                torch.cuda.synchronize(d)
            while len(_scratch) > SCRATCH_PROGRAMS:
                _scratch.popitem(last=False)
        return hit[1], hit[2]


def release_scratch():
    """Free the device staging buffers of the host path (after the device
    has finished the calls that may still use them)."""
    torch = _torch()
    with _scratch_lock:
        if _scratch:
            for d in {k[1] for k in _scratch}:
                torch.cuda.synchronize(d)
            _scratch.clear()


def _execute_host(program: GpuProgram, input_buf, out=None, stream=None, blocking=True, max_device_bytes=None):
    torch = _torch()
    if not torch.cuda.is_available():
        raise VpgError("no CUDA device: the permutation runs only on the GPU (no CPU fallback)")
    lay = program.layout
    as_tensor = isinstance(input_buf, torch.Tensor)
    if as_tensor:
        host = input_buf.contiguous().reshape(-1)
        if host.numel() * host.element_size() != program.nbytes:
            raise LayoutError(f"input holds {host.numel()} elements, program expects {program.num_elements}")
        hbytes = host.view(torch.uint8)
    else:
        if isinstance(input_buf, (bytes, bytearray, memoryview)):
            data = np.frombuffer(input_buf, dtype=np.uint8)
        else:
            data = np.ascontiguousarray(input_buf).reshape(-1).view(np.uint8)
        if data.size != program.nbytes:
            raise LayoutError(f"input holds {data.size // lay.elem_width} elements, "
                              f"program expects {program.num_elements}")
        hbytes = torch.from_numpy(data.copy() if not data.flags.writeable else data)
    dev = torch.device("cuda", torch.cuda.current_device())
    need = 2 * program.nbytes
    if max_device_bytes is None and (_scratch is None or (id(program), dev.index) not in _scratch):
        free = torch.cuda.mem_get_info(dev)[0]
        if need > 0.9 * free:
            max_device_bytes = int(0.5 * free)
    if max_device_bytes is not None and max_device_bytes < need and program.num_elements:
        return _execute_host_bounded(torch, program, hbytes, input_buf, out, stream, dev, int(max_device_bytes))
    d_in, d_out = _host_scratch(torch, program, dev)
    if not blocking and (out is None or not as_tensor or not hbytes.is_pinned() or not out.is_pinned()):
        raise LayoutError("blocking=False needs a pinned CPU tensor input and a pinned `out`")
    if out is None:
        # always pinned: a D2H copy into pageable memory returns only when it
        # completes, which would serialise the chunked pipeline
        h_out = torch.empty(program.nbytes, dtype=torch.uint8, pin_memory=True)
    else:
        h_out = out.reshape(-1).view(torch.uint8)
    if program.num_elements:
        st = torch.cuda.current_stream(dev) if stream is None else stream
        fn = _lib.lib().vpg_permute_host if blocking else _lib.lib().vpg_permute_host_async
        status = fn(
            program.handle, ctypes.c_void_p(hbytes.data_ptr()), ctypes.c_void_p(h_out.data_ptr()),
            ctypes.c_void_p(d_in.data_ptr()), ctypes.c_void_p(d_out.data_ptr()),
            ctypes.c_void_p(st.cuda_stream))
        _check(status, "permute_host")
    if as_tensor:
        if out is not None:
            return out
        res = h_out.view(input_buf.dtype)
        if input_buf.element_size() != program.layout.elem_width:
            return res                                  # opaque bytes: flat
        return res.reshape(program.out_layout.shape_outer_first())
    return h_out.numpy().view(lay.dtype)


def _execute_host_bounded(torch, program, hbytes, input_buf, out, stream, dev, scratch_bytes):
    """Host permutation through a bounded device scratch (vpg_permute_host_bounded)."""
    as_tensor = isinstance(input_buf, torch.Tensor)
    if out is None:
        h_out = torch.empty(program.nbytes, dtype=torch.uint8, pin_memory=hbytes.is_pinned())
    else:
        h_out = out.reshape(-1).view(torch.uint8)
    scratch = torch.empty(scratch_bytes, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream(dev) if stream is None else stream
    status = _lib.lib().vpg_permute_host_bounded(
        program.handle, ctypes.c_void_p(hbytes.data_ptr()), ctypes.c_void_p(h_out.data_ptr()),
        ctypes.c_void_p(scratch.data_ptr()), ctypes.c_size_t(scratch_bytes), ctypes.c_void_p(st.cuda_stream))
    _check(status, "permute_host_bounded")
    del scratch
    if as_tensor:
        if out is not None:
            return out
        res = h_out.view(input_buf.dtype)
        if input_buf.element_size() != program.layout.elem_width:
            return res                                  # opaque bytes: flat
        return res.reshape(program.out_layout.shape_outer_first())
    return h_out.numpy().view(program.layout.dtype)


# ------------------------------------------------------------------ permute
def permute(x, axes, out=None, stream=None):
    """``x.permute(axes).contiguous()`` on the GPU through libvpgpu.so.

    ``x`` is a CUDA tensor, contiguous or a permuted view of contiguous
    memory; ``axes`` use the torch/numpy convention (BASELINE.json's configs
    are stated this way)."""
    torch = _torch()
    if not isinstance(x, torch.Tensor) or not x.is_cuda:
        raise LayoutError("permute needs a CUDA tensor (no CPU fallback)")
    axes = tuple(int(a) for a in axes)
    if len(axes) != x.dim():
        raise LayoutError(f"axes {axes} do not match tensor rank {x.dim()}")
    if x.numel() == 0:                       # nothing to move
        shape = tuple(x.shape[a] for a in axes)
        return torch.empty(shape, dtype=x.dtype, device=x.device) if out is None else out
    if x.dim() == 0:
        res = permute(x.reshape(1), (0,), stream=stream).reshape(())
        return res if out is None else out.copy_(res)
    if not x.is_contiguous():
        x, axes = _dense_base(torch, x, axes)
    layout = TensorLayout.from_shape(tuple(x.shape), x.element_size())
    prog = build_program(layout, from_numpy_convention(axes))
    return execute_device(prog, x, out=out, stream=stream)


def _dense_base(torch, x, axes):
    """A non-contiguous ``x`` that is a permuted view of dense memory
    (``y.permute(p)``, ``y.transpose(i, j)``, ``y.mT``) is permuted from its
    dense base with the composed axes: still one kernel, no copy.  Other
    strided views raise LayoutError."""
    dims = list(range(x.dim()))
    # dense order: descending stride (size-1 dims anywhere; ties keep order)
    order = sorted(dims, key=lambda d: (-x.stride(d) if x.shape[d] > 1 else 0, d))
    order = [d for d in order if x.shape[d] > 1] + [d for d in order if x.shape[d] == 1]
    expect = 1
    for d in reversed(order):
        if x.shape[d] > 1 and x.stride(d) != expect:
            raise LayoutError("input must be contiguous or a permuted view of contiguous memory")
        expect *= x.shape[d]
    base = x.as_strided([x.shape[d] for d in order], _dense_strides([x.shape[d] for d in order]))
    if not base.is_contiguous():
        raise LayoutError("input must be contiguous or a permuted view of contiguous memory")
    pos = {d: i for i, d in enumerate(order)}            # view dim d is base dim pos[d]
    return base, tuple(pos[a] for a in axes)


def _dense_strides(shape):
    st, acc = [], 1
    for n in reversed(shape):
        st.append(acc)
        acc *= n
    return list(reversed(st))
