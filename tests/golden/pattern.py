"""Deterministic golden input pattern (no RNG, reproducible anywhere).

Word i is ``(i + 1) * K mod 2**(8*elem)`` with an odd multiplier K, so every
position holds a distinct word and the output digest pins the permutation
exactly.  The 8-byte pattern uses the full 64 bits (SURVEY.md §4 notes the
reference's own 8-byte test data leaves the high half zero).
"""

from __future__ import annotations

import numpy as np

_K = {1: 0x9D, 2: 0x9E37, 4: 0x9E3779B1, 8: 0x9E3779B97F4A7C15}


def golden_pattern(n: int, elem: int) -> np.ndarray:
    i = np.arange(1, n + 1, dtype=np.uint64)
    if elem == 16:
        lo = i * np.uint64(_K[8])
        hi = (i ^ np.uint64(0xA5A5A5A5A5A5A5A5)) * np.uint64(0xC2B2AE3D27D4EB4F)
        out = np.empty((n, 2), dtype=np.uint64)
        out[:, 0] = lo
        out[:, 1] = hi
        return out.reshape(-1).view(np.dtype([("lo", "<u8"), ("hi", "<u8")]))
    with np.errstate(over="ignore"):
        v = i * np.uint64(_K[elem])
    return v.astype({1: np.uint8, 2: np.uint16, 4: np.uint32, 8: np.uint64}[elem])
