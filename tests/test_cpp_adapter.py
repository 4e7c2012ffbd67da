"""The C++ drop-in (include/wrng_gpu/wallace.hpp) compiled against the C ABI
and run through the reference's own WallaceState scenarios."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1004_3114_b200")


def build(tmp_path):
    exe = tmp_path / "test_adapter"
    subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_adapter.cpp"), "-L", PKG,
                    "-l:libwrng_gpu.so", f"-Wl,-rpath,{PKG}", "-o", str(exe)], check=True)
    return exe


def test_adapter_compiles(tmp_path):
    assert build(tmp_path).exists()


@pytest.mark.gpu
def test_adapter_runs_reference_scenarios(tmp_path):
    exe = build(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
