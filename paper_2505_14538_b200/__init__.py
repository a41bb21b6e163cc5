"""B200-native (sm_100a) hot path of SWIFT's SPHENIX SPH solver (arXiv 2505.14538).

The product is libsph.so (C-ABI in include/sph.h); `binding` is a thin ctypes layer.
"""
from .binding import (  # noqa: F401
    Config,
    Context,
    FIELDS,
    LoopbackGroup,
    SphError,
    default_config,
    lib,
    nccl_unique_id,
    slab_lo,
    slab_mask,
)

__all__ = ["Context", "Config", "FIELDS", "LoopbackGroup", "SphError", "default_config", "lib", "nccl_unique_id",
           "slab_lo", "slab_mask"]
