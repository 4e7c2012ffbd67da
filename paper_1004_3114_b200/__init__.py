"""B200-native Wallace normal generator (Brent's RANN4, arXiv 1004.3114).

The hot path — pool regeneration passes and the exposed output stream — runs
in hand-written sm_100a kernels (csrc/*.cu, built into libwrng_gpu.so) behind the C ABI in
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
    UniformState,
    WallaceState,
    chi2_sf,
    chi2_target,
    plan_segments,
    regenerate,
    rotation_from_t,
    rotation_from_uniform,
    select_pass_params,
    device_anderson_darling,
    device_autocorr,
    device_moments,
    device_uv_chi2,
    lfg_words,
    resident_pools,
    method_fill,
    validate,
)

__all__ = [
    "CorruptedStateError", "CudaError", "MalformedStateError", "PassParams", "Pool",
    "Rotation2", "ScaleMode", "StateErrorKind", "WallaceConfig", "WallaceState",
    "device_moments", "lfg_words", "device_uv_chi2", "device_autocorr", "chi2_sf", "validate",
    "method_fill", "device_anderson_darling", "resident_pools", "UniformState", "chi2_target", "rotation_from_t", "rotation_from_uniform",
    "select_pass_params", "plan_segments", "regenerate",
]
