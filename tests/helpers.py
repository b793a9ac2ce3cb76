"""Shared test helpers (tests only)."""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden", "golden.json")

_golden = None


def golden():
    global _golden
    if _golden is None:
        with open(GOLDEN) as f:
            _golden = json.load(f)
    return _golden


def sha256(arr) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr).view(np.uint8).tobytes()).hexdigest()


def gpu_permute_bytes(dims, sigma, elem, data: np.ndarray, force=None, merge=True, jit=None):
    """Run the GPU path on raw words; returns raw output bytes as uint8."""
    import torch

    from paper_2506_03686_b200 import PermutationMap, TensorLayout, build_program
    from paper_2506_03686_b200.api import execute_device

    raw = np.ascontiguousarray(data).reshape(-1).view(np.uint8)
    x = torch.from_numpy(raw.copy()).cuda()
    prog = build_program(TensorLayout(tuple(dims), elem), PermutationMap(tuple(sigma)),
                         force=force, merge=merge, jit=jit)
    y = execute_device(prog, x)
    return y.cpu().numpy().reshape(-1), prog
