"""ctypes binding of libwrng_gpu.so (the C ABI in include/wrng_gpu.h).

The product path has exactly one implementation: the sm_100a kernels in
csrc/*.cu (libwrng_gpu.so).  If the shared library is missing this module raises at
import time — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("WRNG_GPU_LIB") or os.path.join(HERE, "libwrng_gpu.so")

# wrng_gpu_status
OK = 0
EINVAL = 1
ECORRUPT = 2
EMALFORMED_BAD_MAGIC = 3
EMALFORMED_VERSION = 4
EMALFORMED_TRUNCATED = 5
EMALFORMED_FIELD_RANGE = 6
ECUDA = 7
ENOMEM = 8
ENODEV = 9

F64, F32 = 0, 1
CHISQ, FIXED = 0, 1
FLAG_INIT_HOST = 1 << 0
FLAG_FORCE_HBM = 1 << 1
FLAG_DRIFT_TREE = 1 << 2


class Config(C.Structure):
    _fields_ = [
        ("pool_exponent", C.c_uint32),
        ("throwaway_f", C.c_uint32),
        ("scale_mode", C.c_uint32),
        ("n_arrays", C.c_uint32),
        ("restart_interval_passes", C.c_uint64),
        ("drift_check_period", C.c_uint64),
        ("seed", C.c_uint64),
        ("stream_id", C.c_uint64),
        ("dtype", C.c_uint32),
        ("pools", C.c_uint32),
        ("device", C.c_int32),
        ("flags", C.c_uint32),
    ]


class Params(C.Structure):
    _fields_ = [
        ("stride", C.c_uint32 * 4),
        ("offset", C.c_uint32 * 4),
        ("variant", C.c_uint32),
        ("pad_", C.c_uint32),
        ("c", C.c_double),
        ("s", C.c_double),
        ("scale", C.c_double),
        ("target_sumsq", C.c_double),
    ]


class Counters(C.Structure):
    _fields_ = [
        ("pass_count", C.c_uint64),
        ("numbers_emitted", C.c_uint64),
        ("avail", C.c_uint64),
        ("active", C.c_uint32),
        ("pool_size", C.c_uint32),
    ]


class Validation(C.Structure):  # wrng_gpu_validation
    _fields_ = [
        ("n", C.c_uint64),
        ("m1", C.c_double), ("m2", C.c_double), ("m3", C.c_double), ("m4", C.c_double),
        ("z1", C.c_double), ("z2", C.c_double), ("z4", C.c_double),
        ("uv_samples", C.c_uint64), ("uv_skipped", C.c_uint64),
        ("k", C.c_uint32), ("dof", C.c_uint32),
        ("u_statistic", C.c_double), ("u_p", C.c_double),
        ("v_statistic", C.c_double), ("v_p", C.c_double),
        ("lag", C.c_uint64),
        ("autocorr", C.c_double),
        ("ad_a2", C.c_double),
        ("ad_n", C.c_uint64),
    ]

VALIDATE_AD = 1 << 0


# Every symbol include/wrng_gpu.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "wrng_gpu_config_default", "wrng_gpu_create", "wrng_gpu_destroy",
    "wrng_gpu_fill_f64", "wrng_gpu_fill_f32", "wrng_gpu_advance_pass",
    "wrng_gpu_refill", "wrng_gpu_drift_check", "wrng_gpu_restart",
    "wrng_gpu_get_config", "wrng_gpu_get_counters", "wrng_gpu_read_pool",
    "wrng_gpu_write_pool", "wrng_gpu_read_uniform", "wrng_gpu_export_state",
    "wrng_gpu_import_state", "wrng_gpu_synchronize", "wrng_gpu_last_error",
    "wrng_gpu_kernel_launches", "wrng_gpu_engine", "wrng_gpu_moments_f32",
    "wrng_gpu_moments_f64", "wrng_gpu_lfg_words", "wrng_gpu_uv_counts", "wrng_gpu_autocorr",
    "wrng_gpu_chi2_sf", "wrng_gpu_validate", "wrng_gpu_method_fill",
    # the reference's free functions on host data (reference_api.cu)
    "wrng_gpu_uniform_seed", "wrng_gpu_sumsq_continue", "wrng_gpu_chi2_target",
    "wrng_gpu_rotation_from_t", "wrng_gpu_rotation_from_uniform", "wrng_gpu_select_pass_params",
    "wrng_gpu_plan_segments", "wrng_gpu_regenerate", "wrng_gpu_box_muller_pair",
    "wrng_gpu_box_muller_next", "wrng_gpu_polar_transform", "wrng_gpu_polar_next",
    "wrng_gpu_normal_fill", "wrng_gpu_to_uv", "wrng_gpu_chi2_bins", "wrng_gpu_moments_host",
    "wrng_gpu_autocorr_host", "wrng_gpu_target_stats",
    "wrng_gpu_validate_ex", "wrng_gpu_anderson_darling", "wrng_gpu_resident_pools",
    "wrng_gpu_write_uniform",
)


class Uniform(C.Structure):  # wrng_gpu_uniform (UniformState, uniform.hpp:16-40)
    _fields_ = [
        ("lag_table", C.c_uint64 * 607),
        ("cursor_r", C.c_uint32),
        ("cursor_s", C.c_uint32),
        ("seed", C.c_uint64),
        ("stream_id", C.c_uint64),
        ("draws", C.c_uint64),
    ]


class Segment(C.Structure):  # wrng_gpu_segment (Segment, wallace.hpp:70-75)
    _fields_ = [("low", C.c_uint32), ("high", C.c_uint32), ("jx", C.c_int64), ("jy", C.c_int64)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            "g.build()'` (make -C paper_1004_3114_b200/csrc). There is no CPU fallback.")
    lib = C.CDLL(LIB_PATH)
    vp, u64, u32, i32, dbl = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int32, C.c_double
    P = C.POINTER
    sig = {
        "wrng_gpu_config_default": (None, [P(Config)]),
        "wrng_gpu_create": (C.c_int, [P(Config), P(vp)]),
        "wrng_gpu_destroy": (None, [vp]),
        "wrng_gpu_fill_f64": (C.c_int, [vp, vp, u64, dbl, dbl, C.c_int, vp]),
        "wrng_gpu_fill_f32": (C.c_int, [vp, vp, u64, dbl, dbl, C.c_int, vp]),
        "wrng_gpu_advance_pass": (C.c_int, [vp, vp]),
        "wrng_gpu_refill": (C.c_int, [vp]),
        "wrng_gpu_drift_check": (C.c_int, [vp]),
        "wrng_gpu_restart": (C.c_int, [vp]),
        "wrng_gpu_get_config": (C.c_int, [vp, P(Config)]),
        "wrng_gpu_get_counters": (C.c_int, [vp, u32, P(Counters)]),
        "wrng_gpu_read_pool": (C.c_int, [vp, u32, vp, P(dbl), P(dbl)]),
        "wrng_gpu_write_pool": (C.c_int, [vp, u32, vp, dbl, dbl]),
        "wrng_gpu_read_uniform": (C.c_int, [vp, u32, vp, P(u32), P(u32), P(u64)]),
        "wrng_gpu_export_state": (C.c_int, [vp, vp, C.c_size_t, P(C.c_size_t)]),
        "wrng_gpu_import_state": (C.c_int, [vp, C.c_size_t, i32, u32, P(vp)]),
        "wrng_gpu_synchronize": (C.c_int, [vp]),
        "wrng_gpu_last_error": (C.c_char_p, [vp]),
        "wrng_gpu_kernel_launches": (u64, [vp]),
        "wrng_gpu_engine": (C.c_char_p, [vp]),
        "wrng_gpu_moments_f32": (C.c_int, [vp, u64, vp, i32, vp]),
        "wrng_gpu_moments_f64": (C.c_int, [vp, u64, vp, i32, vp]),
        "wrng_gpu_lfg_words": (C.c_int, [u64, u64, u32, u64, vp, i32]),
        "wrng_gpu_uv_counts": (C.c_int, [vp, i32, u64, u32, vp, vp, P(u64), i32, vp]),
        "wrng_gpu_autocorr": (C.c_int, [vp, i32, u64, u64, P(dbl), i32, vp]),
        "wrng_gpu_chi2_sf": (dbl, [dbl, u32]),
        "wrng_gpu_validate": (C.c_int, [vp, u64, u32, u64, vp, vp, P(Validation)]),
        "wrng_gpu_method_fill": (C.c_int, [i32, u64, u64, u32, vp, i32, u64, dbl, dbl, i32, i32,
                                           vp]),
        "wrng_gpu_uniform_seed": (None, [P(Uniform), u64, u64]),
        "wrng_gpu_sumsq_continue": (dbl, [dbl, vp, u64]),
        "wrng_gpu_chi2_target": (dbl, [dbl, u32]),
        "wrng_gpu_rotation_from_t": (None, [dbl, u32, P(dbl), P(dbl)]),
        "wrng_gpu_rotation_from_uniform": (None, [P(Uniform), P(dbl), P(dbl)]),
        "wrng_gpu_select_pass_params": (C.c_int, [P(Uniform), u32, u32, u32, dbl, dbl,
                                                  P(Params)]),
        "wrng_gpu_plan_segments": (C.c_int, [P(Params), u32, vp, u32, P(u32)]),
        "wrng_gpu_regenerate": (C.c_int, [vp, vp, u32, u32, P(Params), P(dbl), i32]),
        "wrng_gpu_box_muller_pair": (C.c_int, [dbl, dbl, P(dbl), P(dbl)]),
        "wrng_gpu_box_muller_next": (None, [P(Uniform), P(dbl), P(dbl)]),
        "wrng_gpu_polar_transform": (None, [dbl, dbl, P(dbl), P(dbl)]),
        "wrng_gpu_polar_next": (None, [P(Uniform), P(dbl), P(dbl)]),
        "wrng_gpu_normal_fill": (None, [i32, P(Uniform), vp, u64, dbl, dbl]),
        "wrng_gpu_to_uv": (None, [dbl, dbl, P(dbl), P(dbl), P(i32)]),
        "wrng_gpu_chi2_bins": (C.c_int, [vp, u64, u32, dbl, dbl, P(dbl)]),
        "wrng_gpu_moments_host": (C.c_int, [vp, u64, vp]),
        "wrng_gpu_autocorr_host": (C.c_int, [vp, u64, u64, P(dbl)]),
        "wrng_gpu_target_stats": (None, [vp, u64, vp]),
        "wrng_gpu_validate_ex": (C.c_int, [vp, u64, u32, u64, u32, vp, vp, P(Validation)]),
        "wrng_gpu_anderson_darling": (C.c_int, [vp, i32, u64, P(dbl), i32, vp]),
        "wrng_gpu_resident_pools": (C.c_int64, [P(Config)]),
        "wrng_gpu_write_uniform": (C.c_int, [vp, u32, vp, u32, u32, u64]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()
