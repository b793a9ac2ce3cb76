"""TEST INFRASTRUCTURE ONLY -- run the reference's own emitted CPU kernels.

Loads ``oracle/_ref/lib<cfg>_<target>.so`` built by ``oracle/build_ref.py``
and calls ``void permute_<hash>(const void *src, void *dst)`` (the C ABI of
emit.py:118-128, 219) through ctypes.  Buffers follow the reference harness
(emit.py:370-396): 64-byte aligned, with ``w * elem`` bytes of writable slack
before and after the data (emit.py:5-8).

Used by tests (full-size parity at BASELINE sizes) and by bench.py's
``--impl reference`` arm / ``cpu_baseline`` leg.  Never by the product.
"""

from __future__ import annotations

import ctypes
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")

__all__ = ["available", "manifest", "host_has_avx512", "RefKernel", "SlackBuffer"]


def manifest() -> dict:
    path = os.path.join(REF_DIR, "manifest.json")
    if not os.path.exists(path):
        return {}
    with open(path) as f:
        return json.load(f)


def host_has_avx512() -> bool:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("flags"):
                    return "avx512f" in line.split(":", 1)[1].split()
    except OSError:
        pass
    return False


def available(cfg: str) -> bool:
    return cfg in manifest()


class SlackBuffer:
    """64-byte aligned byte buffer with ``slack`` bytes before/after the data."""

    def __init__(self, nbytes: int, slack: int):
        self.nbytes = nbytes
        self.slack = slack
        total = nbytes + 2 * slack + 128
        self._raw = np.zeros(total, dtype=np.uint8)
        base = self._raw.ctypes.data
        pad = (-(base + slack)) % 64            # data start 64-byte aligned
        self.offset = pad + slack
        self.data = self._raw[self.offset:self.offset + nbytes]

    @property
    def ptr(self) -> int:
        return self._raw.ctypes.data + self.offset

    def view(self, dtype) -> np.ndarray:
        return self.data.view(dtype)


class RefKernel:
    """The reference's emitted kernel for one BASELINE config."""

    def __init__(self, cfg: str, target: str | None = None):
        man = manifest()
        if cfg not in man:
            raise RuntimeError(f"no reference kernel for {cfg}; run python oracle/build_ref.py")
        entry = man[cfg]
        if target is None:
            target = "x86-avx" if host_has_avx512() else "scalar"
        if target not in entry["targets"]:
            raise RuntimeError(f"no {target} kernel for {cfg}")
        t = entry["targets"][target]
        self.cfg = cfg
        self.target = target
        self.entry = entry
        self.elem_bytes = int(entry["elem_bytes"])
        self.slack = int(entry["slack_bytes"])
        self.numel = int(np.prod(entry["shape"]))
        self.nbytes = self.numel * self.elem_bytes
        self._lib = ctypes.CDLL(os.path.join(REF_DIR, t["so"]))
        self.fn = getattr(self._lib, t["symbol"])
        self.fn.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        self.fn.restype = None

    def alloc(self) -> SlackBuffer:
        return SlackBuffer(self.nbytes, self.slack)

    def run_ptr(self, src_ptr: int, dst_ptr: int) -> None:
        self.fn(src_ptr, dst_ptr)

    def __call__(self, data: np.ndarray) -> np.ndarray:
        """Permute raw words of ``data`` (any dtype of the right byte size)."""
        raw = np.ascontiguousarray(data).reshape(-1).view(np.uint8)
        if raw.size != self.nbytes:
            raise ValueError(f"expected {self.nbytes} bytes, got {raw.size}")
        src = self.alloc()
        dst = self.alloc()
        src.data[:] = raw
        self.fn(src.ptr, dst.ptr)
        return dst.data.copy()
