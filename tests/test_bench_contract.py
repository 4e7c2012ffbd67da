"""bench.py's JSON contract: the reference arm (CPU only, runs here) and our
arm (needs the GPU) print one line with the keys the driver reads."""
import json
import os
import subprocess
import sys

import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                       capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_reference_arm_line():
    d = run_bench("--impl", "reference", "--steps", "1", "--warmup", "0",
                  "--ref-sample-per-thread", str(1 << 16))
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "dtype", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["bench_loop"]["value"] > 0
    assert "workload" in d["config"]


@pytest.mark.gpu
def test_our_arm_line():
    d = run_bench("--total", str(1 << 28), "--steps", "3", "--warmup", "3", "--e2e-sample",
                  str(1 << 22), "--e2e-steps", "1", "--cpu-seconds", "0.2")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "roofline", "gpu_launches", "clocks", "e2e", "cpu_baseline"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["value"] > 0
    assert d["gpu_launches"] >= 3  # one fill kernel per step
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] <= 1.2
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == (1 << 22) * 4
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])


def test_gpus_flag_fails_loudly_without_enough_devices():
    """`bench.py --gpus N` outside torchrun launches N ranks itself; with
    fewer devices than N it must fail, not measure one GPU (CPU here)."""
    import torch

    want = max(2, torch.cuda.device_count() + 1)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(want),
                        "--steps", "1", "--warmup", "0"], cwd=ROOT, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 2
    assert f"needs {want} CUDA devices" in r.stderr
    assert not [l for l in r.stdout.splitlines() if l.startswith("{")]
