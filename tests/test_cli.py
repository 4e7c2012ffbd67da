"""The wrng-gpu CLI (tools/wrng_gpu_cli.cpp): the reference CLI's gen /
stream / test / bench subcommands (tools/main.cpp) on the B200 backend,
built against the drop-in header.  Usage errors run on CPU; the rest on
the GPU, compared with the unmodified reference library's stream and state
bytes (oracle/_ref)."""
import os
import subprocess

import numpy as np
import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tools", "wrng-gpu")


@pytest.fixture(scope="module")
def cli():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tools")], check=True)
    return BIN


def run(cli, *args, **kw):
    return subprocess.run([cli, *args], capture_output=True, timeout=600, **kw)


@pytest.mark.parametrize("args", [
    [], ["bogus"], ["gen", "--pool-exponent", "7"], ["gen", "--pool-exponent", "21"],
    ["gen", "--f", "0"], ["gen", "--sigma", "-1"], ["gen", "--format", "xml"],
    ["gen", "--methods", "wallace"], ["bench", "--methods", "wallace,foo"],
    ["test", "--suite", "nope"], ["gen", "--count"], ["stream", "--count", "5"],
])
def test_usage_errors_exit_2(cli, args):
    # main.cpp:27-30: usage error -> 2, before touching the device
    assert run(cli, *args).returncode == 2


@pytest.mark.gpu
@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_gen_f64le_equals_reference_stream(cli):
    r = run(cli, "gen", "--count", "50001", "--format", "f64le", "--seed", "12345", "--f", "1",
            "--pool-exponent", "12", "--mu", "0.25", "--sigma", "2")
    assert r.returncode == 0, r.stderr
    got = np.frombuffer(r.stdout, dtype="<f8")
    want = O.RefState(pool_exponent=12, throwaway_f=1, seed=12345).fill(50001, 0.25, 2.0)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


@pytest.mark.gpu
def test_gen_text_format(cli):
    r = run(cli, "gen", "--count", "7", "--seed", "3", text=True)
    assert r.returncode == 0
    vals = [float(x) for x in r.stdout.split()]
    want = O.OracleState(pool_exponent=10, throwaway_f=3, seed=3).fill(7)
    assert [f"{v:.17g}" for v in want] == r.stdout.split() and np.array_equal(vals, want)


@pytest.mark.gpu
@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_gen_state_file_resumes_like_reference(cli, tmp_path):
    sf = str(tmp_path / "state.wrng")
    a = run(cli, "gen", "--count", "1000", "--format", "f64le", "--state-file", sf, "--seed", "9")
    b = run(cli, "gen", "--count", "1500", "--format", "f64le", "--state-file", sf)
    assert a.returncode == 0 and b.returncode == 0
    got = np.frombuffer(a.stdout + b.stdout, dtype="<f8")
    ref = O.RefState(pool_exponent=10, throwaway_f=3, seed=9)
    assert np.array_equal(got, ref.fill(2500))
    assert open(sf, "rb").read() == ref.save_state()  # "WRNG" v1, byte-identical
    with open(sf, "r+b") as fh:
        fh.write(b"XXXX")
    assert run(cli, "gen", "--count", "1", "--state-file", sf).returncode == 3


@pytest.mark.gpu
def test_stream_until_consumer_closes(cli):
    p = subprocess.Popen([cli, "stream", "--seed", "5"], stdout=subprocess.PIPE)
    head = p.stdout.read(8 * 20000)
    p.stdout.close()
    assert p.wait(timeout=120) == 0
    want = O.OracleState(pool_exponent=10, throwaway_f=3, seed=5).fill(20000)
    assert np.array_equal(np.frombuffer(head, dtype="<f8"), want)


@pytest.mark.gpu
@pytest.mark.parametrize("suite,samples", [("uniformity", "400000"), ("moments", "2000000"),
                                           ("sumsq", "3000")])
def test_test_suites_pass(cli, suite, samples):
    r = run(cli, "test", "--suite", suite, "--samples", samples, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "result=PASS" in r.stdout and f"{suite}." in r.stdout


@pytest.mark.gpu
def test_bench_prints_every_method(cli):
    r = run(cli, "bench", "--methods", "wallace-gpu,polar,boxmuller-gpu", "--seconds", "0.2",
            "--fp32", "--n-arrays", "4", "--f", "1", text=True)
    assert r.returncode == 0, r.stderr
    for m in ("wallace-gpu", "polar-gpu", "boxmuller-gpu"):
        line = [x for x in r.stdout.splitlines() if x.startswith(f"bench.{m}.ns_per_value=")]
        assert line and float(line[0].split("=")[1]) > 0
