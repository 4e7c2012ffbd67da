"""CPU tests of the drop-in boundary: libwrng_gpu.so loads, exports every
symbol include/wrng_gpu.h declares, and fails cleanly without a GPU."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "wrng_gpu.h")
LIB = os.path.join(ROOT, "paper_1004_3114_b200", "libwrng_gpu.so")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(wrng_gpu_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared()
    for must in ("wrng_gpu_create", "wrng_gpu_fill_f64", "wrng_gpu_fill_f32",
                 "wrng_gpu_advance_pass", "wrng_gpu_refill", "wrng_gpu_drift_check",
                 "wrng_gpu_export_state", "wrng_gpu_import_state", "wrng_gpu_destroy",
                 "wrng_gpu_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB), "build first: make -C paper_1004_3114_b200/csrc"
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r" T (wrng_gpu_\w+)", out))
    missing = [n for n in declared() if n not in exported]
    assert not missing, missing
    from paper_1004_3114_b200 import _lib

    assert set(_lib.EXPORTS) == set(declared())


def test_library_is_sm100a_cubin():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_config_default_matches_reference_defaults():
    from paper_1004_3114_b200 import _lib

    c = _lib.Config()
    _lib.lib.wrng_gpu_config_default(C.byref(c))
    # WallaceConfig defaults (wallace.hpp:57-65)
    assert (c.pool_exponent, c.throwaway_f, c.scale_mode, c.restart_interval_passes,
            c.drift_check_period, c.seed, c.stream_id) == (10, 3, 0, 0, 64, 0, 0)
    assert (c.n_arrays, c.dtype, c.pools, c.device, c.flags) == (2, 0, 1, 0, 0)


def test_invalid_config_is_einval_before_device_access():
    from paper_1004_3114_b200 import _lib

    c = _lib.Config()
    _lib.lib.wrng_gpu_config_default(C.byref(c))
    h = C.c_void_p()
    for field, value in (("pool_exponent", 7), ("pool_exponent", 21), ("throwaway_f", 0),
                         ("n_arrays", 3), ("dtype", 2), ("pools", 0)):
        bad = _lib.Config.from_buffer_copy(c)
        setattr(bad, field, value)
        assert _lib.lib.wrng_gpu_create(C.byref(bad), C.byref(h)) == _lib.EINVAL
    bad = _lib.Config.from_buffer_copy(c)
    bad.throwaway_f, bad.restart_interval_passes = 3, 3
    assert _lib.lib.wrng_gpu_create(C.byref(bad), C.byref(h)) == _lib.EINVAL


def test_malformed_state_rejected_without_device():
    from paper_1004_3114_b200 import _lib

    h = C.c_void_p()
    buf = (C.c_uint8 * 8)(*b"NOPE\x01\x00\x00\x00")
    assert _lib.lib.wrng_gpu_import_state(buf, 8, 0, 0, C.byref(h)) == _lib.EMALFORMED_BAD_MAGIC
    buf = (C.c_uint8 * 3)(*b"GNR")
    assert _lib.lib.wrng_gpu_import_state(buf, 3, 0, 0, C.byref(h)) == _lib.EMALFORMED_TRUNCATED
    buf = (C.c_uint8 * 8)(*(b"GNRW" + b"\x09\x00\x00\x00"))
    assert _lib.lib.wrng_gpu_import_state(buf, 8, 0, 0, C.byref(h)) == _lib.EMALFORMED_VERSION


@pytest.mark.skipif(os.environ.get("CUDA_VISIBLE_DEVICES") is None and
                    subprocess.run(["nvidia-smi"], capture_output=True).returncode == 0,
                    reason="a GPU is present")
def test_create_without_gpu_fails_loudly():
    from paper_1004_3114_b200 import _lib

    c = _lib.Config()
    _lib.lib.wrng_gpu_config_default(C.byref(c))
    h = C.c_void_p()
    assert _lib.lib.wrng_gpu_create(C.byref(c), C.byref(h)) == _lib.ENODEV
    assert not h.value


def test_product_package_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_1004_3114_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in text.replace("oracle/", "").lower() or f == "__init__.py", f
