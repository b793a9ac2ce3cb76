"""Seeded synthetic inputs for the BASELINE.json configurations.

BASELINE.json names no public dataset; these generators stand in for the
reference's measurement inputs with the stated shapes, dtypes and value
distributions.  Inputs are generated in blocks of 2**22
elements with ``np.random.default_rng([seed, block])`` so any block can be
regenerated independently and the same bytes reach the CPU and the GPU.

Shapes and axes use the NumPy/torch convention (outer-to-inner,
``out = x.permute(axes)``), as BASELINE.json does.
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

BLOCK = 1 << 22

__all__ = ["Workload", "CONFIGS", "cfg5_axes", "make_input", "make_input_slice", "get_config"]


def cfg5_axes(seed: int = 0, rank: int = 28) -> tuple[int, ...]:
    """First ``rng.permutation(28)`` from ``default_rng(seed)`` whose last
    axis moves (BASELINE.json configs[4])."""
    rng = np.random.default_rng(seed)
    while True:
        p = rng.permutation(rank)
        if p[rank - 1] != rank - 1:
            return tuple(int(x) for x in p)


@dataclass(frozen=True)
class Workload:
    key: str
    title: str
    shape: tuple[int, ...]
    axes: tuple[int, ...]
    dtype: str          # numpy dtype name
    dist: str           # "uniform" ([-1,1)) or "normal"

    @property
    def elem_bytes(self) -> int:
        return np.dtype(self.dtype).itemsize

    @property
    def numel(self) -> int:
        n = 1
        for d in self.shape:
            n *= d
        return n

    @property
    def algorithmic_bytes(self) -> int:
        """One read + one write per element."""
        return 2 * self.numel * self.elem_bytes

    @property
    def out_shape(self) -> tuple[int, ...]:
        return tuple(self.shape[a] for a in self.axes)


CONFIGS: dict[str, Workload] = {
    "cfg1": Workload("cfg1", "2-D transpose f32 (4096,4096) perm (1,0)",
                     (4096, 4096), (1, 0), "float32", "uniform"),
    "cfg2": Workload("cfg2", "NCHW->NHWC f32 (32,64,56,56) perm (0,2,3,1)",
                     (32, 64, 56, 56), (0, 2, 3, 1), "float32", "normal"),
    "cfg3": Workload("cfg3", "misaligned 6-D f32 (17,9,13,15,11,27) perm (5,2,0,4,1,3)",
                     (17, 9, 13, 15, 11, 27), (5, 2, 0, 4, 1, 3), "float32", "uniform"),
    "cfg4": Workload("cfg4", "stride-1-preserved f64 (128,64,32,512) perm (2,0,1,3)",
                     (128, 64, 32, 512), (2, 0, 1, 3), "float64", "normal"),
    "cfg5": Workload("cfg5", "rank-28 all-2 complex64 (2,)*28, seeded random perm",
                     (2,) * 28, cfg5_axes(0), "complex64", "normal"),
}


def get_config(key: str) -> Workload:
    if key not in CONFIGS:
        raise KeyError(f"unknown config {key!r}; expected one of {sorted(CONFIGS)}")
    return CONFIGS[key]


def _fill_block(flat: np.ndarray, wl: Workload, seed: int, b: int) -> None:
    lo = b * BLOCK
    hi = min(flat.size, lo + BLOCK)
    m = hi - lo
    rng = np.random.default_rng([seed, b])
    if wl.dtype == "complex64":
        flat[lo:hi] = rng.standard_normal(2 * m, dtype=np.float32).view(np.complex64)
    elif wl.dist == "uniform":
        flat[lo:hi] = rng.random(m, dtype=np.dtype(wl.dtype)) * 2 - 1
    else:
        flat[lo:hi] = rng.standard_normal(m, dtype=np.dtype(wl.dtype))


def make_input(wl: Workload | str, seed: int = 0, threads: int = 8) -> np.ndarray:
    """Seeded input tensor (outer-first shape) for a workload."""
    if isinstance(wl, str):
        wl = get_config(wl)
    out = np.empty(wl.numel, dtype=np.dtype(wl.dtype))
    nblocks = -(-wl.numel // BLOCK)
    if nblocks == 1 or threads <= 1:
        for b in range(nblocks):
            _fill_block(out, wl, seed, b)
    else:
        with ThreadPoolExecutor(max_workers=threads) as ex:
            list(ex.map(lambda b: _fill_block(out, wl, seed, b), range(nblocks)))
    return out.reshape(wl.shape)


def make_input_slice(wl: Workload | str, lo: int, hi: int, seed: int = 0) -> np.ndarray:
    """Elements [lo, hi) of the flattened seeded input (each rank of the
    sharded mode regenerates only its own shard)."""
    if isinstance(wl, str):
        wl = get_config(wl)
    out = np.empty(hi - lo, dtype=np.dtype(wl.dtype))
    for b in range(lo // BLOCK, -(-hi // BLOCK)):
        b0 = b * BLOCK
        m = min(BLOCK, wl.numel - b0)
        blk = np.empty(m, dtype=out.dtype)
        rng = np.random.default_rng([seed, b])
        if wl.dtype == "complex64":
            blk[:] = rng.standard_normal(2 * m, dtype=np.float32).view(np.complex64)
        elif wl.dist == "uniform":
            blk[:] = rng.random(m, dtype=np.dtype(wl.dtype)) * 2 - 1
        else:
            blk[:] = rng.standard_normal(m, dtype=np.dtype(wl.dtype))
        s0, s1 = max(lo, b0), min(hi, b0 + m)
        out[s0 - lo:s1 - lo] = blk[s0 - b0:s1 - b0]
    return out
