"""The reference's OWN test suites, run unchanged.

/root/reference/proj/tests/{test_uniform, test_reference, test_wallace_core,
test_wallace_state, test_serialize, test_stats}.cpp (55 doctest cases) and
acceptance.cpp (the 11 shipping criteria) are compiled
from where they lie, by tests/cpp/Makefile, with an original
doctest-compatible shim (tests/cpp/shim/doctest.h):

  * against the reference library itself (oracle/_ref) — proves the shim
    runs the suites faithfully (CPU, no GPU needed);
  * against the B200 drop-in (include/wrng_gpu/compat/wrng/*.hpp ->
    include/wrng_gpu/*.hpp over libwrng_gpu.so) — the reference's callers
    and tests, unmodified, on the GPU.

The binaries are built in this container (build()) and travel to the GPU
box; nothing here reads /root/reference at run time.
"""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
B = os.path.join(ROOT, "tests", "cpp", "_build")


def run_suite(name, timeout=900):
    exe = os.path.join(B, name)
    if not os.path.exists(exe):
        pytest.fail(f"{exe} not built (tests/cpp/Makefile needs /root/reference at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=timeout)
    print(r.stdout[-6000:])
    print(r.stderr[-6000:])
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed", r.stdout)
    assert m, r.stdout + r.stderr
    return r.returncode, int(m.group(1)), int(m.group(2)), r.stdout


def _ref_built():
    return os.path.exists(os.path.join(B, "ref_unit_ref"))


@pytest.mark.skipif(not _ref_built(), reason="reference suites not built here")
def test_shim_runs_reference_unit_suite_on_reference_library():
    rc, total, passed, _ = run_suite("ref_unit_ref", timeout=300)
    assert rc == 0 and total == passed == 55


@pytest.mark.skipif(not _ref_built(), reason="reference suites not built here")
def test_shim_runs_reference_acceptance_on_reference_library():
    rc, total, passed, out = run_suite("ref_acceptance_ref", timeout=300)
    assert rc == 0 and total == passed == 11
    assert out.count("[PASS]") == 16 and "[FAIL]" not in out


@pytest.mark.gpu
def test_reference_unit_suite_on_gpu_dropin():
    rc, total, passed, _ = run_suite("ref_unit_gpu")
    assert rc == 0 and total == passed == 55


@pytest.mark.gpu
def test_reference_acceptance_on_gpu_dropin():
    rc, total, passed, out = run_suite("ref_acceptance_gpu")
    assert rc == 0 and total == passed == 11
    assert out.count("[PASS]") == 16 and "[FAIL]" not in out
