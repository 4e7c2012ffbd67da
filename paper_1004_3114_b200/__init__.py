"""B200-native Wallace normal generator (Brent's RANN4, arXiv 1004.3114).

The hot path — pool regeneration passes and the exposed output stream — runs
in hand-written sm_100a kernels (csrc/kernels.cu) behind the C ABI in
include/wrng_gpu.h.  This package is the Python host mirror of the
reference's generator interface (proj/include/wrng/wallace.hpp).
"""
from .wallace import (  # noqa: F401
    CorruptedStateError,
    CudaError,
    MalformedStateError,
    PassParams,
    Pool,
    Rotation2,
    ScaleMode,
    StateErrorKind,
    WallaceConfig,
    WallaceState,
    device_moments,
    lfg_words,
)

__all__ = [
    "CorruptedStateError", "CudaError", "MalformedStateError", "PassParams", "Pool",
    "Rotation2", "ScaleMode", "StateErrorKind", "WallaceConfig", "WallaceState",
    "device_moments", "lfg_words",
]
