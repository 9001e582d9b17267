"""B200-native electrostatic PIC hot path (arxiv 2605.05469, FFT-PIC Landau damping).

The compute path is libpic.so (CUDA, sm_100a) behind the C ABI of
include/pic.h; ``_binding`` is its thin ctypes binding.
"""
from ._binding import (  # noqa: F401
    PicError,
    PifSolver,
    PIF_STAGES,
    Simulation,
    STAGES,
    default_params,
    domain,
    lib,
    nccl_unique_id,
    owner_ranks,
    slab,
    slab_select,
    workspace_bytes,
)
from ._build import build_lib  # noqa: F401
