"""B200-native general N-D tensor permutation (GenTT, arXiv 2506.03686).

Drop-in for the permutation hot path of the reference package ``vecperm``:
same layout/map types and conventions, ``build_program`` / ``execute``
plan-and-run API, plus ``permute(x, axes)`` and the sharded multi-GPU
``permute_sharded``.  Kernels are hand-written for sm_100a and live in
``libvpgpu.so`` behind the C ABI of ``include/vpgpu.h``.
"""

from .core import (
    SUPPORTED_ELEM_WIDTHS,
    LayoutError,
    PermutationMap,
    TensorLayout,
    compute_strides,
    dtype_for_width,
    from_numpy_convention,
    permuted_layout,
    to_numpy_convention,
)
from .api import (
    GpuProgram,
    GpuTarget,
    VpgError,
    build_program,
    emit_source,
    execute,
    format_plan,
    jit_compile,
    merge_dimensions,
    permute,
    program_cache_clear,
    autotune,
    release_scratch,
)

__version__ = "0.1.0"

__all__ = [
    "SUPPORTED_ELEM_WIDTHS",
    "LayoutError",
    "PermutationMap",
    "TensorLayout",
    "compute_strides",
    "dtype_for_width",
    "from_numpy_convention",
    "permuted_layout",
    "to_numpy_convention",
    "GpuProgram",
    "GpuTarget",
    "VpgError",
    "build_program",
    "execute",
    "emit_source",
    "format_plan",
    "jit_compile",
    "merge_dimensions",
    "permute",
    "program_cache_clear",
    "autotune",
    "release_scratch",
]
