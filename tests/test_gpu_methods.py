"""GPU Box-Muller / polar baselines (reference.cpp:9-63)
against the oracle restatement (pinned to the reference library in
tests/test_oracle.py) and the live reference.

Bars: f64 math is the reference's expression sequence with CUDA libm, so
values agree to TOL64 = 1e-12 normwise (|gpu - ref| <= 1e-12 * max(1, |ref|));
the polar accept/reject sequence is exact arithmetic, so a single wrong
decision would shift every later value and fail the tolerance.  fp32
outputs of f64 math: TOL32 = 1e-6 relative.  fp32 math (the throughput
variant): 1e-3 absolute.
"""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

TOL64 = 1e-12
TOL32 = 1e-6


@pytest.fixture(scope="module")
def W():
    import paper_1004_3114_b200 as W

    return W


def close(a, b, tol):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    err = np.abs(a - b) / np.maximum(1.0, np.abs(b))
    assert float(err.max()) <= tol, f"max normwise error {err.max():.3e} > {tol}"


def run(W, method, count, pools, dtype="f64", f64_math=True, mu=0.0, sigma=1.0, seed=5,
        stream=3):
    import torch

    t = torch.empty(count, dtype=torch.float64 if dtype == "f64" else torch.float32,
                    device="cuda")
    W.method_fill(method, t, seed, stream, pools, mu, sigma, f64_math)
    torch.cuda.synchronize()
    return t.cpu().numpy()


@pytest.mark.parametrize("method", ["boxmuller", "polar"])
@pytest.mark.parametrize("pools,count", [(1, 10001), (5, 5 * 3000 + 3), (148, 148 * 513)])
def test_f64_math_matches_oracle(W, method, pools, count):
    got = run(W, method, count, pools)
    want = O.method_bank_fill(method, 5, 3, pools, count)
    close(got, want, TOL64)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("method", ["boxmuller", "polar"])
def test_matches_live_reference(W, method):
    got = run(W, method, 20001, 1, mu=0.5, sigma=2.0)
    u = O.RefUniform(5, 3)
    want = (u.box_muller_fill if method == "boxmuller" else u.polar_fill)(20001, 0.5, 2.0)
    close(got, want, TOL64)


@pytest.mark.parametrize("method", ["boxmuller", "polar"])
def test_f32_outputs(W, method):
    got = run(W, method, 7 * 4001, 7, dtype="f32")
    want = O.method_bank_fill(method, 5, 3, 7, 7 * 4001)
    close(got, want.astype(np.float32), TOL32)
    fast = run(W, method, 7 * 4001, 7, dtype="f32", f64_math=False)
    assert float(np.max(np.abs(fast.astype(np.float64) - want))) <= 1e-3


def test_edge_cases(W):
    import torch

    t = torch.zeros(1, dtype=torch.float64, device="cuda")
    W.method_fill("polar", t, 1, 0, 1)  # odd length: the first pair's x
    torch.cuda.synchronize()
    close(t.cpu().numpy(), O.method_bank_fill("polar", 1, 0, 1, 1), TOL64)
    e = torch.zeros(0, dtype=torch.float64, device="cuda")
    W.method_fill("boxmuller", e, 1, 0, 1)  # empty: no-op
    with pytest.raises(ValueError):
        W.method_fill("boxmuller", t, 1, 0, 1, sigma=-1.0)
    # more pools than values: empty streams write nothing
    t3 = torch.full((3,), 9.0, dtype=torch.float64, device="cuda")
    W.method_fill("boxmuller", t3, 2, 0, 8)
    torch.cuda.synchronize()
    close(t3.cpu().numpy(), O.method_bank_fill("boxmuller", 2, 0, 8, 3), TOL64)
